"""Write profiles/ppmm_traffic.json (bench.py's roofline.traffic) from an ncu
DRAM capture of one c4 (8-part) PPMM launch (profile.sh step 3), with the
sha256 of the kernel source it was taken from.

    python profiles/update_traffic.py profiles/<tag>_ppmm_dram_c4.csv
"""
import csv
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    src = Path(sys.argv[1])
    rows = [r for r in csv.reader(src.open()) if len(r) > 14 and r[0] != "ID"]
    val = {r[12]: float(r[14]) for r in rows if "ppmm_i8_sm100_kernel<1, 4, 0>" in r[4]}
    parts = 8
    rd, wr = val["dram__bytes_read.sum"], val["dram__bytes_write.sum"]
    P, M, N, K = 24, 1 << 14, 992, 24576
    algo = P * 2 * M * K + P * 2 * N * K + P * N * M * 2  # DB planes + query planes + uint16 outputs
    out = {"bytes_per_part": (rd + wr) / parts, "dram_read_per_part": rd / parts, "dram_write_per_part": wr / parts,
           "algorithmic_bytes_per_part": algo, "launch_ms_under_ncu": val["gpu__time_duration.sum"] / 1e6,
           "source": f"{src.relative_to(ROOT) if src.is_absolute() else src}: ncu dram__bytes_read.sum / "
                     "dram__bytes_write.sum of one c4 (8-part) launch, divided by 8",
           "kernel_source_sha256": hashlib.sha256(
               (ROOT / "paper_2601_17561_b200" / "csrc" / "ppmm_gemm.cu").read_bytes()).hexdigest()}
    (ROOT / "profiles" / "ppmm_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
