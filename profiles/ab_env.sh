#!/bin/bash
# A/B of an environment knob on one box (alternating runs): bash profiles/ab_env.sh "VAR=1" "VAR2=..." -- [power_probe args]
VARS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do VARS+=("$1"); shift; done
shift
for rep in 1 2; do
  for V in "${VARS[@]}"; do
    env $V timeout 300 python profiles/power_probe.py "$@" | sed "s|^{|{\"env\": \"$V\", |"
  done
done
