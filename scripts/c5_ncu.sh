#!/bin/bash
# C5 ablation under ncu (run on the GPU box): FA and VFA at (d, Bc) in {64,128}^2, C2 shape.
# Per kernel: pipe utilisation and the per-opcode instruction mix; summarise here with
# scripts/c5_ncu_summary.py. Numbers printed under ncu are not bench values.
set -u
OUT=${1:-gpurun_out/c5}
mkdir -p "$OUT"
M=gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum
M=$M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__issue_active.avg.pct_of_peak_sustained_active,sass__inst_executed_per_opcode
for d in 128 64; do
  for bc in 128 64; do
    nl=1; [ "$bc" = 64 ] && nl=2
    for v in fa vfa; do
      tag=${v}_d${d}_b${bc}
      timeout 300 ncu --metrics "$M" --clock-control none -k regex:vfa_fwd_kernel -s 1 -c 1 -f -o "$OUT/$tag" \
        python scripts/profile_step.py --variant $v --head-dim $d --k-block $bc --n-local $nl \
        --stats-out "$OUT/$tag.json" > "$OUT/$tag.log" 2>&1 || echo "FAILED $tag"
    done
  done
done
ls "$OUT"
