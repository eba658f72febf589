# shared-C K1: row parameters loaded one stage ahead (default) vs at the stage (build/libbase_shared.so)
for lib in default build/libbase_shared.so; do
  echo "== $lib"
  if [ "$lib" = default ]; then python tools/lockstep_ab.py 2>&1 | grep -E "ms per batch|evals" | grep lockstep-decoupled;
  else MDOT_LIB=$lib python tools/lockstep_ab.py 2>&1 | grep -E "ms per batch|evals" | grep lockstep-decoupled; fi
done
