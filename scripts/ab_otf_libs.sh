#!/bin/bash
# A/B of K2 library variants (build/lib*.so from scripts/build_variant.py) on
# the config-5 evaluation: scripts/ab_otf_libs.sh out.log lib1 lib2 ...
out=$1; shift
: > "$out"
for lib in "$@"; do
  echo "== $lib" >> "$out"
  if [ "$lib" = base ]; then python scripts/otf_recipe_ab.py dot diff >> "$out" 2>&1
  else MDOT_LIB=build/lib$lib.so python scripts/otf_recipe_ab.py dot diff >> "$out" 2>&1; fi
done
