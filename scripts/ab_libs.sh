#!/bin/bash
# A/B of library builds on the bench workload: prints K1 in-solve mean, time-to-eps, evaluations.
for L in "$@"; do
  if [ "$L" = base ]; then unset MDOT_LIB; else export MDOT_LIB=$PWD/build/lib$L.so; fi
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --adaptive-leg 0 --adaptive-gamma-leg 0 --no-config5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
print('$L', 'k1_us=%.2f'%d['roofline']['mean_launch_us'], 'frac=%.3f'%d['roofline']['frac'], 'tte_ms=%.1f'%d['ms_per_step'], 'evals=%d'%d['evaluations_per_solve'], 'l1=%.3g'%d['solve']['l1_final'], 'cost=%.12g'%d['solve']['cost_unrounded'], 'stages', d['slot_stage_us'], 'clk', d['clocks']['sm_mhz'])"
done
