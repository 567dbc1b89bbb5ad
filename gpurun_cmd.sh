mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/plain.log 2>&1 && cat gpurun_out/plain.log | tail -1 | cut -c1-300 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:modup_ip32 -s 8 -c 1 -o gpurun_out/modup_ip $CMD > gpurun_out/ncu_a.log 2>&1; echo ncu_a rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:vecmat_lazy_mont -s 2 -c 1 -o gpurun_out/vecmat_lazy $CMD > gpurun_out/ncu_b.log 2>&1; echo ncu_b rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 800 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_c.log 2>&1; echo ncu_c rc=$?
