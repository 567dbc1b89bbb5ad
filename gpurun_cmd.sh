mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scheme.py -q -m gpu -k "small" 2>&1 | tail -15
