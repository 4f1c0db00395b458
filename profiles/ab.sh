#!/bin/bash
# A/B of PPMM library variants on one box (alternating runs to cancel clock drift).
#   bash profiles/ab.sh <out.jsonl> <variant.so|default> ... -- [power_probe args]
OUT=$1; shift
LIBS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do LIBS+=("$1"); shift; done
shift
for rep in 1 2; do
  for L in "${LIBS[@]}"; do
    if [ "$L" = default ]; then unset IRL_B200_LIB; else export IRL_B200_LIB=$PWD/$L; fi
    timeout 300 python profiles/power_probe.py "$@" | sed "s|^{|{\"lib\": \"$L\", |" >> $OUT
  done
done
unset IRL_B200_LIB
cat $OUT
