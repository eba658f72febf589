# k_finalize_multi blocks per SM (MDOT_FIN_MULTI_PER_SM; 4 = the earlier rule, 8 = default) on the lockstep batch
for ps in 1 2 4; do
  echo "== per_sm $ps"
  MDOT_FIN_MULTI_PER_SM=$ps python tools/lockstep_ab.py 2>&1 | grep "ms per batch" | grep lockstep-decoupled
done
