"""The C++ host mirror (irislab_b200/modmat.hpp) driven by the reference's own
unit-suite cases (tests/cpp/test_modmat_b200.cpp restates
proj/tests/test_modmat.cpp). Built here on CPU; executed on a B200."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2601_17561_b200"
BIN = ROOT / "build" / "test_modmat_b200"
BIN_IRIS = ROOT / "build" / "test_iris_b200"
BIN_CCMM = ROOT / "build" / "test_ccmm_b200"


def _build_driver(src, out):
    cmd = ["/usr/bin/g++", "-O2", "-std=c++17", f"-I{PKG / 'host'}", str(src), "-o", str(out), f"-L{PKG}",
           "-lirl_b200", f"-L{ROOT / 'oracle'}", "-l:libirl_oracle.so", f"-Wl,-rpath,{PKG}",
           f"-Wl,-rpath,{ROOT / 'oracle'}"]
    subprocess.run(cmd, check=True)


@pytest.fixture(scope="module")
def iris_binary(binary):
    _build_driver(ROOT / "tests/cpp/test_iris_b200.cpp", BIN_IRIS)
    return BIN_IRIS


@pytest.fixture(scope="module")
def binary():
    from paper_2601_17561_b200 import build
    if not (PKG / "libirl_b200.so").exists():
        build.build()
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    BIN.parent.mkdir(exist_ok=True)
    cmd = ["/usr/bin/g++", "-O2", "-std=c++17", f"-I{PKG / 'host'}", str(ROOT / "tests/cpp/test_modmat_b200.cpp"),
           "-o", str(BIN), f"-L{PKG}", "-lirl_b200", f"-L{ROOT / 'oracle'}", "-l:libirl_oracle.so",
           f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{ROOT / 'oracle'}"]
    subprocess.run(cmd, check=True)
    return BIN


def test_cpp_mirror_builds_and_links(binary):
    assert binary.exists()
    syms = subprocess.run(["nm", "-DC", str(PKG / "libirl_b200.so")], capture_output=True, text=True).stdout
    for fn in ["irislab::modmat::gemm_mod_psq", "irislab::modmat::gemm_mod_Q", "irislab::modmat::digit_decompose",
               "irislab::modmat::small_gemm", "irislab::modmat::save_big_matrix"]:
        assert fn in syms


@pytest.mark.gpu
def test_cpp_mirror_reference_unit_suite(binary):
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600, cwd=ROOT / "build")
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_cpp_iris_mirror_builds(iris_binary):
    assert iris_binary.exists()
    syms = subprocess.run(["nm", "-DC", str(PKG / "libirl_b200.so")], capture_output=True, text=True).stdout
    for fn in ["irislab::iris::score", "irislab::iris::match_db_reference", "irislab::iris::inner_and_overlap"]:
        assert fn in syms


@pytest.mark.gpu
def test_cpp_iris_mirror_reference_unit_suite(iris_binary):
    r = subprocess.run([str(iris_binary)], capture_output=True, text=True, timeout=600, cwd=ROOT / "build")
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.fixture(scope="module")
def ccmm_binary(binary):
    _build_driver(ROOT / "tests/cpp/test_ccmm_b200.cpp", BIN_CCMM)
    return BIN_CCMM


def test_cpp_ccmm_mirror_builds(ccmm_binary):
    assert ccmm_binary.exists()
    syms = subprocess.run(["nm", "-DC", str(PKG / "libirl_b200.so")], capture_output=True, text=True).stdout
    for fn in ["irislab::emu::ccmm_twin_product", "irislab::b200::CcmmEngine::run", "irislab::b200::CcmmGroup::run"]:
        assert fn in syms


@pytest.mark.gpu
def test_cpp_ccmm_mirror_reference_case(ccmm_binary):
    r = subprocess.run([str(ccmm_binary)], capture_output=True, text=True, timeout=600, cwd=ROOT / "build")
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_cpp_costmodel_mirror_reference_vectors():
    """irislab_b200/costmodel.hpp against the reference's test_costmodel.cpp
    vectors (36/18 GiB, 62 packed cts, 37 clusters at 2^22) and the B200
    residency plan (a whole 8-part cluster per 180 GB GPU). Header-only: CPU."""
    out = ROOT / "build" / "test_costmodel_b200"
    out.parent.mkdir(exist_ok=True)
    subprocess.run(["/usr/bin/g++", "-O2", "-std=c++17", f"-I{PKG / 'host'}",
                    str(ROOT / "tests/cpp/test_costmodel_b200.cpp"), "-o", str(out)], check=True)
    r = subprocess.run([str(out)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "0 failed" in r.stdout, r.stdout
