mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ring.py tests/test_gpu_cnn.py tests/test_gpu_scheme.py -q -m gpu -k "small or cnn or lazy or ntt" 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench17.json 2> gpurun_out/bench17.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench17.json'))
print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['hbm_frac'])
print({k:v['ms_per_step'] for k,v in list(d['breakdown'].items())[:10]})"
