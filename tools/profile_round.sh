#!/bin/bash
# ncu evidence for one round (run under gpurun): launch list of one cfg2
# factorization + one `ncu --set full` capture per top kernel family.
# usage: bash tools/profile_round.sh r04   -> gpurun_out/<tag>_*.{csv,ncu-rep}
# (FFB_JACOBI_NOFUSE: ncu cannot replay the fused cooperative+cluster Jacobi
#  launch faithfully; FFB_GRAPHS=0: one node per launch in the list)
tag=${1:-r04}
export FFB_JACOBI_NOFUSE=1 FFB_GRAPHS=0
one="python tools/one_factorization.py --workload cfg2 --warmup 1"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches_cfg2.csv $one > gpurun_out/${tag}_ncu_list.log 2>&1
full="ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -c 1"
$full -k "regex:gemm_f64_kernel<\(int\)64, \(int\)144" -o gpurun_out/${tag}_k13 $one > gpurun_out/${tag}_ncu_k13.log 2>&1
$full -k "regex:gemm_f64_kernel<\(int\)80, \(int\)64, \(int\)16, \(int\)40, \(int\)32, \(bool\)1" -o gpurun_out/${tag}_sketch $one > gpurun_out/${tag}_ncu_sketch.log 2>&1
$full -k "regex:jacobi_kernel" -o gpurun_out/${tag}_jacobi $one > gpurun_out/${tag}_ncu_jacobi.log 2>&1
$full -k "regex:panel_qr_kernel" -o gpurun_out/${tag}_panel $one > gpurun_out/${tag}_ncu_panel.log 2>&1
$full -k "regex:pivots_kernel" -o gpurun_out/${tag}_pivots $one > gpurun_out/${tag}_ncu_pivots.log 2>&1
ls -la gpurun_out/${tag}_*
