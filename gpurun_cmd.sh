mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scheme.py tests/test_gpu_edges.py tests/test_gpu_configs.py -q -m gpu -k "encrypt or empty or ragged or cfg3" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
