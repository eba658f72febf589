# shared-C K1 consumer: 4-row group loop unrolled 1 (shipped before) / 4 / 8, lockstep batch 16 x n = 4096
for lib in build/libshu4.so build/libshu8.so; do
  echo "== $lib"
  MDOT_LIB=$lib python tools/lockstep_ab.py 2>&1 | grep -E "ms per batch|evals" | grep lockstep-decoupled
done
