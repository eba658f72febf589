for rep in 1 2; do
  MDOT_LIB=$PWD/build/lib_head.so timeout 120 python scripts/time_batch.py 2>&1 | head -3 | sed 's/^/head /'
  timeout 120 python scripts/time_batch.py 2>&1 | head -3 | sed 's/^/fast /'
done
