# K8 tile loop: 4-row steps unrolled 1 (shipped) vs 2, config 2 (64 pairs), two rounds
for round in 1 2; do
  python tools/k8_ab_once.py
  MDOT_LIB=build/libk8u2.so python tools/k8_ab_once.py
done
