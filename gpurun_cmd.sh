mkdir -p gpurun_out
for B in 128 256 512 1024; do
timeout 600 python bench.py --steps 3 --warmup 3 --batch $B --no-cpu-baseline --no-extra > gpurun_out/bench_b$B.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_b$B.json'))
print($B, round(d['value']), round(d['e2e']['value']), d['roofline']['kernel'], d['roofline']['frac'])"
done
