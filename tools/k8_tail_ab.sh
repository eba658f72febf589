# K8 balanced last row block (MDOT_K8_TAIL1) A/B on config 2: default library vs build/libk8tail0.so, two rounds
for round in 1 2; do
  python tools/k8_ab_once.py
  MDOT_LIB=build/libk8tail0.so python tools/k8_ab_once.py
done
