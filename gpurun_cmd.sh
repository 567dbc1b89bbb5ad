mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -q -m gpu 2>&1 | tail -25
