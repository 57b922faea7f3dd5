# A/B timing of two builds of the library on the same box:
#   bash tools/ab_bench.sh <config> <lib A> [<lib B> = in-tree build] [rounds]
cfg=$1; A=$2; B=${3:-paper_2501_07145_b200/_lib/libsigkern_b200.so}; R=${4:-2}
for r in $(seq $R); do
  for lib in $A $B; do
    v=$(SK_LIB_OVERRIDE=$lib python bench.py --config $cfg --no-cpu --e2e-steps 1 2>/dev/null | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['roofline']['frac'],4))")
    echo "$cfg $(basename $lib): $v"
  done
done
