#!/usr/bin/env bash
# Round-end evidence under gpurun (1 GPU):
#   1. bench.py (the driver's default command) -> gpurun_out/<tag>_bench.json
#   2. the ncu launch list of the same workload (greedy matrix pinned)
#   3. ncu --set full of the dominant kernel (-k regex $TOPK) at the bench size
# usage: bash tools/profile_bench.sh <tag> [top-kernel-regex]
set -u
tag=${1:-cur}
topk=${2:-conv_stack}
out=gpurun_out
mkdir -p $out
if [ -z "${MATRIX:-}" ]; then
  timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
  cat $out/${tag}_bench.json
  matrix=$(python -c "import json;print(','.join(map(str,json.load(open('$out/${tag}_bench.json'))['config']['matrix_A2'][0])))")
else
  matrix=$MATRIX  # bench already run: profile this matrix only
fi
echo "matrix $matrix"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/${tag}_launches.csv python bench.py --matrix $matrix --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > $out/${tag}_launches.log 2>&1 || echo "launch list failed"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$topk" -s 3 -c 1 \
  -o $out/${tag}_top -f python bench.py --matrix $matrix --steps 1 --warmup 3 --no-cpu-baseline \
  --no-e2e > $out/${tag}_top.log 2>&1 || echo "ncu top failed"
