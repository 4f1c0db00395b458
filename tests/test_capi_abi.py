"""CPU-side checks of the drop-in boundary: libirl_b200.so builds for sm_100a,
loads, and exports every symbol include/irl_capi.h declares; context creation
fails loudly (no CPU fallback) when there is no sm_100 device."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "irl_capi.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(irl_[A-Za-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_17561_b200 import build, capi
    if not capi.LIB_PATH.exists():
        build.build()
    return capi.lib()


def test_header_and_binding_table_agree():
    from paper_2601_17561_b200 import capi
    assert declared_functions() == sorted(capi.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib._name)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\b(irl_[A-Za-z0-9_]+)\b", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_library_is_sm100a_cuda(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib._name)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(lib._name)], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass  # tcgen05.mma kind::i8
    assert "UTCOMMA" in sass  # tcgen05.mma kind::mxf4.block_scale (iris products on FP4)
    assert "UTMALDG" in sass  # TMA tile loads
    assert "LDTM" in sass     # tcgen05.ld (TMEM -> registers)


def test_pure_host_helpers(lib):
    import ctypes as C
    import numpy as np
    from paper_2601_17561_b200 import capi
    assert lib.irl_abi_version() == 1
    p = np.zeros(64, np.uint32)
    e = np.zeros(64, np.uint32)
    n = lib.irl_paper_basis(capi.ptr(p, capi.u32p), capi.ptr(e, capi.u32p), 64)
    assert n == 24 and p[0] == 127 and p[23] == 251 and (e[:n] == 2).all()
    buf = np.zeros(64, np.uint8)
    w = lib.irl_basis_Q_bytes(capi.ptr(p, capi.u32p), capi.ptr(e, capi.u32p), n, capi.ptr(buf, capi.u8p), 64)
    q = 1
    for v in p[:n]:
        q *= int(v) ** 2
    assert w == 46 and int.from_bytes(bytes(buf[:w]), "little") == q
    assert lib.irl_status_string(3) == b"AccumulationOverflowRisk"


def test_host_generator_matches_oracle(lib):
    import oracle_lib as ol
    for args in [(1, 0, 0, 0, 0, 16129), (77, 255, 23, 4095, 24575, 63001), (2**63 + 5, 7, 3, 12345, 9, 127 * 127)]:
        assert lib.irl_synth_residue(*args) == ol.oracle().orc_synth_residue(*args)


def test_no_device_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import ctypes as C
    h = C.c_void_p()
    assert lib.irl_ctx_create(0, C.byref(h)) == 8  # IRL_ERR_NO_DEVICE
    from paper_2601_17561_b200 import modmat
    with pytest.raises(modmat.DeviceError):
        modmat.Context(0)


def test_fold_params_struct_layout_matches_header(tmp_path):
    """capi.FoldParams (ctypes) has the size and field offsets the C compiler
    gives irl_fold_params."""
    import ctypes as C

    from paper_2601_17561_b200 import capi
    fields = [f for f, _ in capi.FoldParams._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "irl_capi.h"\nint main(void) {\n'
                   '    printf("%zu", sizeof(irl_fold_params));\n' +
                   "".join(f'    printf(" %zu", offsetof(irl_fold_params, {f}));\n' for f in fields) +
                   "    return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["/usr/bin/gcc", "-std=c11", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == C.sizeof(capi.FoldParams)
    assert got[1:] == [getattr(capi.FoldParams, f).offset for f in fields]


def test_ppmm_psq_kernels_keep_everything_in_registers(lib):
    """The mod-p^2 PPMM kernels (mode 0) must not touch local memory: a stack
    frame for the TMEM accumulator arrays (seen once in r2, after a change
    lengthened a live range in the epilogue) doubled the kernel's DRAM writes."""
    sass = subprocess.run(["cuobjdump", "-sass", str(lib._name)], capture_output=True, text=True).stdout
    funcs = sass.split("Function : ")
    psq = [f for f in funcs if "ppmm_i8_sm100_kernelILi" in f.split("\n", 1)[0] and "ELi0EEE" in f.split("\n", 1)[0]]
    assert len(psq) >= 4
    for f in psq:
        body = f.split("\n", 1)[1]
        assert " STL" not in body and " LDL" not in body, f.split("\n", 1)[0]
