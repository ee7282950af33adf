#!/bin/bash
# A/B of the sparse group passes' sampling geometry (EPSM_MULTI_GEOM=q:sk forces it for every
# group pass): usage tools/geom_sweep.sh "256:32 64:16" "4:16 8:16 16:16 8:8"
for C in $1; do
  echo "== $C default: $(timeout 60 python tools/code_ab.py $C 5 2>&1 | tail -1)"
  for G in $2; do
    echo "   geom $G: $(EPSM_MULTI_GEOM=$G timeout 60 python tools/code_ab.py $C 5 2>&1 | tail -1)"
  done
done
