#!/bin/bash
# usage: tools/hot_lines.sh <src.csv> <mangled kernel> [top]  -- per-source-line share of instructions / stall samples
python "$(dirname "$0")/sass_lines.py" "$1" /tmp/cub/epsm.sm_100a.cubin "$2" "${3:-30}" > /tmp/hot.txt
python - <<'PY'
src=open('/root/repo/paper_1209_6449_b200/csrc/epsm_kernels.cuh').read().split('\n')
for l in open('/tmp/hot.txt'):
    p=l.split()
    if p and p[0].startswith('epsm_kernels.cuh:'):
        n=int(p[0].split(':')[1]); print(l.rstrip()[:70], '|', src[n-1].strip()[:80])
    else: print(l.rstrip())
PY
