mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scheme.py tests/test_gpu_cnn.py -q -m gpu -k "bsgs or cnn" 2>&1 | tail -15
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench21.json 2> gpurun_out/bench21.err; echo bench rc=$?
tail -2 gpurun_out/bench21.err
python -c "
import json; d=json.load(open('gpurun_out/bench21.json'))
print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['hbm_frac'])
print({k:v['ms_per_step'] for k,v in list(d['breakdown'].items())[:12]})"
