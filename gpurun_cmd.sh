set -x
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final5.txt 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final5.txt 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench42.json 2> gpurun_out/bench42.err; echo "bench rc=$?"
python bench.py > gpurun_out/bench42b.json 2> gpurun_out/bench42b.err; echo "bench2 rc=$?"
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench42_plain.json 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_v42.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_list42.log 2>&1; echo "ncu list rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench42_ref.json 2> gpurun_out/bench42_ref.err; echo "ref rc=$?"
tail -2 gpurun_out/pytest_gpu_final5.txt; tail -1 gpurun_out/smoke_final5.txt
