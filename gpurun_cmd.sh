mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench19.json 2> gpurun_out/bench19.err; echo bench rc=$?
tail -3 gpurun_out/bench19.err
python -c "
import json; d=json.load(open('gpurun_out/bench19.json'))
print(d['value'], d['e2e']['value']); print(json.dumps(d['extra']['ops_table45'])); print(d['extra']['communication_cfg4'])"
