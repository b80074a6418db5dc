#!/bin/bash
# Build kPolyPairs variants in-tree and time each (bench numbers; not under ncu).
set -u
cd "$(dirname "$0")/.."
for p in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -cudart static \
    -DVFA_POLY_PAIRS=$p -o paper_2604_12798_b200/libvfa_b200_p$p.so paper_2604_12798_b200/csrc/vfa_fwd.cu &
done
wait
for p in "$@"; do
  echo "poly_pairs=$p"
  VFA_B200_LIB=$PWD/paper_2604_12798_b200/libvfa_b200_p$p.so timeout 300 python bench.py --no-cpu --no-e2e --steps 20 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print({k:(v['attn_kernel_tflops'] if isinstance(v,dict) else v) for k,v in d['ablation'].items()}, d['clocks'])"
done
