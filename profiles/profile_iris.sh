#!/bin/bash
# ncu --set full of the FP4 iris match main launch (query columns on M, 4x1
# clusters) at the paper's scale, under gpurun (1 GPU):  bash profiles/profile_iris.sh <tag>
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"ppmm_i8_sm100_kernel<\(int\)4" -s 2 -c 1 -o $OUT/iris_full_$TAG -f \
  python profiles/iris_match_ab.py --reps 1 > $OUT/iris_full_$TAG.log 2>&1
$NCU -i $OUT/iris_full_$TAG.ncu-rep --page raw --csv > $OUT/iris_full_$TAG.csv 2>&1
python - "$OUT/iris_full_$TAG.csv" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__cluster_dim_x",
        "launch__registers_per_thread"]
for w in want:
    for i, n in enumerate(h):
        if n == w or n.endswith(w):
            print(f"{n} | {u[i]} | {v[i]}")
            break
PY
