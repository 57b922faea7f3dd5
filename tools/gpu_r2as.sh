timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
bash tools/gpu_r2ad.sh > /dev/null 2>&1
for c in c3 c1 c2 c4 c5; do python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), round(d['e2e']['value']), d['clocks']['reasons'])"; done
head -12 gpurun_out/r2_c3_bench_launches.txt
