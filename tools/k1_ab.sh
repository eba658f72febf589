# bench/k1bench.cu A/B builds (build/k1b_*): product K1 at n = 4096 (C L2-resident, evict_last) and n = 16384,
# plus the harness's read-only / TMA-ring streams at n = 4096 and 2048
for v in base; do
  echo "== $v"
  K1B_KEEP=1 K1B_TM=256 ./build/k1b_$v 4096 400 q
  K1B_KEEP=1 K1B_TM=256 ./build/k1b_$v 2048 400 q
  K1B_KEEP=1 K1B_TM=512 ./build/k1b_$v 8192 100 q
done
