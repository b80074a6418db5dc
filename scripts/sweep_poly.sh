#!/bin/bash
# Build VFA_POLY_PAIRS variants in-tree (libvfa_b200_p<N>.so) and A/B-time them interleaved
# in one process (scripts/ab.py; experiment numbers, not bench values).
#   scripts/sweep_poly.sh 0 1 2 3
set -u
cd "$(dirname "$0")/.."
for p in "$@"; do
  python -c "import sys; sys.path.insert(0, '.'); from paper_2604_12798_b200 import build; print(build.build(defines=('p' + sys.argv[1], ['-DVFA_POLY_PAIRS=' + sys.argv[1]])))" "$p"
done
libs=""
for p in "$@"; do libs="$libs p$p=paper_2604_12798_b200/libvfa_b200_p$p.so"; done
for v in vfa fa; do timeout 300 python scripts/ab.py --variant $v $libs; done
