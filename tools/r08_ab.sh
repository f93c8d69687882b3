#!/bin/bash
# A/B timing of library variants: bash tools/r08_ab.sh <log> <cfgs...> -- <libs...>
set -u
LOG=$1; shift
CFGS=(); while [ "$1" != "--" ]; do CFGS+=("$1"); shift; done; shift
mkdir -p gpurun_out/r08
for cfg in "${CFGS[@]}"; do
  for lib in "$@"; do
    SW_B200_LIB=$lib timeout 600 python tools/quick_time.py $cfg >> gpurun_out/r08/$LOG 2>&1
  done
done
grep -E "median|fwd kernel|rev swept|lib:" gpurun_out/r08/$LOG
