#!/bin/bash
# A/B timing of library variants: bash tools/r09_ab.sh <log> <cfgs...> -- <libs...>  (parity of each lib on c2[0:3000] first)
set -u
LOG=$1; shift
CFGS=(); while [ "$1" != "--" ]; do CFGS+=("$1"); shift; done; shift
mkdir -p gpurun_out/r09
for lib in "$@"; do
  SW_B200_LIB=$lib timeout 300 python tools/band_repro.py c2 3000 0 x >> gpurun_out/r09/$LOG 2>&1
  echo "parity lib: $lib" >> gpurun_out/r09/$LOG
done
for cfg in "${CFGS[@]}"; do
  for lib in "$@"; do
    SW_B200_LIB=$lib timeout 600 python tools/quick_time.py $cfg >> gpurun_out/r09/$LOG 2>&1
  done
done
grep -E "mismatches [1-9]|parity lib|median|fwd kernel|rev swept|lib:" gpurun_out/r09/$LOG
