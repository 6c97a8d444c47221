python bench.py --no-also --no-cpu-baseline > gpurun_out/bq.json 2>gpurun_out/bq.err
python -c "
import json; d=json.load(open('gpurun_out/bq.json')); print(round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,4) for k, v in (d.get('stage_ms') or {}).items()})"
