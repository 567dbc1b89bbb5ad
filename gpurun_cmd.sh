mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests/test_gpu_cnn.py -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 3 --warmup 3 --batch 128 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
