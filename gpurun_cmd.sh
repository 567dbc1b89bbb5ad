mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r01_final.json 2> gpurun_out/bench_r01_final.err; echo bench rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:vecmat_lazy_mont -s 2 -c 1 -o gpurun_out/vecmat_lazy3 $CMD > gpurun_out/ncu_a.log 2>&1; echo ncu_a rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:modup_ip32 -s 8 -c 1 -o gpurun_out/modup_ip3 $CMD > gpurun_out/ncu_b.log 2>&1; echo ncu_b rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 800 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_c.log 2>&1; echo ncu_c rc=$?
