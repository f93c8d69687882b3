#!/bin/bash
set -u
LOG=$1; shift
mkdir -p gpurun_out/r09
for lib in "$@"; do
  echo "lib $lib" >> gpurun_out/r09/$LOG
  SW_B200_LIB=$lib timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "cooperative or reverse_band or c5 or c3_protein or stripe" 2>&1 | tail -1 >> gpurun_out/r09/$LOG
done
for cfg in c3 c5; do for lib in "$@"; do
  SW_B200_LIB=$lib timeout 600 python tools/quick_time.py $cfg >> gpurun_out/r09/$LOG 2>&1
done; done
grep -E "^lib|passed|failed|median|stages|lib:" gpurun_out/r09/$LOG
