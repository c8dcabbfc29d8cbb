#!/bin/bash
# A/B of one environment switch: inversion ubench + bench value, both arms
# alternating twice (same box).  Usage: bash tools/gpu_ab.sh TAG VAR=off_value
set -u
TAG=$1; OFF=$2
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
run() { echo "== $*" >> "$OUT/log.txt"; "$@" >> "$OUT/log.txt" 2>&1; echo "rc=$?" >> "$OUT/log.txt"; }
[ -n "${TESTS:-}" ] && run timeout 900 python -m pytest $TESTS -x -q
one() { echo -n "$* : " >> "$OUT/res.txt"; env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],4), round(d['phases']['inversion']['ms'],4), d['check']['inverse_residual_max'])" >> "$OUT/res.txt"; }
for i in 1 2; do
  env PF_X=1 timeout 300 python tools/ubench_inv.py 4096:2 "4096:2,1024:10" 1024:8 2048:4 >> "$OUT/ubench_on.txt" 2>&1
  env $OFF timeout 300 python tools/ubench_inv.py 4096:2 "4096:2,1024:10" 1024:8 2048:4 >> "$OUT/ubench_off.txt" 2>&1
  one PF_X=1
  one $OFF
done
echo finished >> "$OUT/log.txt"
