mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_scheme.py -q -m gpu -k "cnn_layers or rescale" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench26_$i.json 2>gpurun_out/bench26.err; python -c "
import json; d=json.load(open('gpurun_out/bench26_$i.json'))
print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])
print({k:v['ms_per_step'] for k,v in list(d['breakdown'].items())[:12]})"; done
