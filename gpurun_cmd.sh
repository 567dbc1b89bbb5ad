mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench11.json 2> gpurun_out/bench11.err; echo bench rc=$?
tail -3 gpurun_out/bench11.err
python -c "
import json; d=json.load(open('gpurun_out/bench11.json'))
print(d['value'], d['e2e']['value']); print(json.dumps(d['extra'], indent=0))"
