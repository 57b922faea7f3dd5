# A/B device time of one config at a reduced N: bash tools/ab_devtime.sh <cfg> <N> <lib A> [<lib B>]
cfg=$1; n=$2; A=$3; B=${4:-paper_2501_07145_b200/_lib/libsigkern_b200.so}
for r in 1 2; do for lib in $A $B; do
  echo "$(basename $lib): $(SK_LIB_OVERRIDE=$lib python tools/devtime.py $cfg $n fp32 3 2>&1 | tail -1)"
done; done
