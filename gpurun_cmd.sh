mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --batch 128 --no-cpu-baseline --no-extra"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:JobKsData -s 40 -c 1 -o gpurun_out/ksdata $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
python scratch/prof_ntt.py 14 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:JobLimbs -s 2 -c 2 -o gpurun_out/ntt14 python scratch/prof_ntt.py 14 > gpurun_out/ncu3.log 2>&1; echo ncu3 rc=$?
ls -la gpurun_out
