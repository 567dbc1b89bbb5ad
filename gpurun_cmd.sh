mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scheme.py tests/test_gpu_cnn.py -q -m gpu -k "lazy or bsgs or cnn_layers" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'])"; done
