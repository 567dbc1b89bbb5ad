timeout 1500 python -m pytest tests/test_gpu_scheme.py -q -m gpu 2>&1 | tail -40
