#!/bin/bash
# bench (headline only) for the base library and each lib_var variant given
for v in base "$@"; do
  if [ $v = base ]; then unset BSG_LIB; else export BSG_LIB=/root/repo/paper_2405_13943_b200/lib_var/libbsgpu_$v.so; fi
  python bench.py --no-also --no-cpu-baseline > gpurun_out/bq_$v.json 2>gpurun_out/bq_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/bq_$v.json')); print('$v', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,4) for k, v in (d.get('stage_ms') or {}).items() if v > 0.05})"
done
