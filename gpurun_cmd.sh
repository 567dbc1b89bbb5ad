mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_scheme.py -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --batch 128 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench2.json'))
print(d['value'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])
print({k:v['ms_per_step'] for k,v in list(d['breakdown'].items())[:6]})
print(d['extra'])"
