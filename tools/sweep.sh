#!/bin/bash
# run bench for the default lib and every variant; one JSON summary line per variant
for v in default $(ls paper_2602_05081_b200/variants/*.so 2>/dev/null) default; do
  if [ "$v" = default ]; then unset GF_LIB; name=default; else export GF_LIB=$PWD/$v; name=$(basename $v .so); fi
  timeout 600 python bench.py --config ${CFG:-2} ${EXTRA} --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],3), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['stage_ms_per_step'].items()})"
done
