#!/usr/bin/env bash
# Every BASELINE.json config on one B200 with the current build (design
# evidence for DESIGN.md §8): gpurun_out/<tag>_cfgN.json, one bench line each.
# usage: bash tools/run_configs.sh <tag>
set -u
tag=${1:-cur}
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${tag}_$c.json 2> gpurun_out/${tag}_$c.err
  python -c "import json;d=json.load(open('gpurun_out/${tag}_$c.json'));print('$c',d['value'],d['ms_per_step'],d['roofline']['kernel'],d['roofline']['frac'],d['e2e']['value'] if d.get('e2e') else None)" || tail -3 gpurun_out/${tag}_$c.err
done
