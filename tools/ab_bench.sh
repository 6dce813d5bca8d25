#!/usr/bin/env bash
# Same-box A/B of two library builds on the cfg2 step (power-capped, like the
# driver's bench): alternates the in-tree library and tools/base_prev/ twice.
# usage: bash tools/ab_bench.sh [extra bench args]
set -u
for i in 1 2; do
  for l in "" base_prev; do
    if [ -n "$l" ]; then
      cp paper_2208_14049_b200/libenserve_b200.so /tmp/lib_new.so
      cp tools/base_prev/libenserve_b200.so paper_2208_14049_b200/libenserve_b200.so
    fi
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --matrix 128,128,128,128 "$@" > /tmp/ab.json 2>/dev/null
    python -c "import json;d=json.load(open('/tmp/ab.json'));print('${l:-new}', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], [round(k['ms'],3) for k in d['roofline']['per_kernel']])"
    if [ -n "$l" ]; then cp /tmp/lib_new.so paper_2208_14049_b200/libenserve_b200.so; fi
  done
done
