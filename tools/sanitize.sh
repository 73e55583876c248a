#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the flag-synchronised
# kernels (run on the GPU box; logs under gpurun_out/sanitize/).
set -u
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
cases=(
  "base::128x128 1"
  "wave64::32x32 64"
  "front:TFB_FRONT_SOLVE=2 TFB_FRONT_MIN_FRONTS=1:128x128 1"
  "split:TFB_FRONT_SOLVE=0 TFB_SPLIT_SOLVE=2:128x128 1"
  "lookahead:TFB_LOOKAHEAD_COLS=64 TFB_LOOKAHEAD_ROOT_COLS=64 TFB_ROOT_DATAFLOW=0:128x128 1"
  "3d::8x8x8 1"
)
for tool in memcheck racecheck synccheck; do
  for c in "${cases[@]}"; do
    tag=${c%%:*}; rest=${c#*:}; envs=${rest%%:*}; args=${rest#*:}
    log="$OUT/${tool}_${tag}.log"
    echo "== $tool $tag ($envs) args=$args" > "$log"
    timeout 900 env $envs $CS --tool $tool --error-exitcode 9 \
      python tools/sanitize_case.py $args >> "$log" 2>&1
    echo "exit=$?" >> "$log"
    tail -3 "$log"
  done
done
