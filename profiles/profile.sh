#!/bin/bash
# ncu evidence for the bench's dominant kernel (run under gpurun, 1 GPU).
#   bash profiles/profile.sh <tag>
# Outputs land in gpurun_out/ (scratch); summaries are copied to profiles/.
set -x
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
BENCH="python bench.py --no-e2e --no-cpu-baseline --no-int8-ref"
# 1) launch list of the bench command (cold-cache, serialised: shares only)
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_$TAG.csv $BENCH --steps 2 --warmup 1 > $OUT/launches_$TAG.log 2>&1
# 2) full capture of one PPMM launch (1 part = one DB slice, c2/c3 geometry)
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ppmm_i8" -s 2 -c 1 \
  -o $OUT/ppmm_full_$TAG -f $BENCH --parts 1 --steps 1 --warmup 1 > $OUT/ppmm_full_$TAG.log 2>&1
# 3) DRAM traffic of the full 8-part launch (single-pass metric group)
timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --kernel-name-base demangled -k regex:"ppmm_i8" -s 2 -c 1 --csv --log-file $OUT/ppmm_dram_$TAG.csv \
  $BENCH --steps 1 --warmup 1 > $OUT/ppmm_dram_$TAG.log 2>&1
ls -la $OUT
