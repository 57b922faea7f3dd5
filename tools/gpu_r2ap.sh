for r in 8 4 2 1; do
  echo "rx $r"; SK_RX_MULTI=$r timeout 300 python tools/devtime.py c5 512 fp32 2 0 nofix | tail -1
done
SK_RX_MULTI=1 timeout 300 python tools/devtime.py L512d4M8 2048 fp32 2 0 nofix | tail -1
