#!/bin/bash
# ncu evidence for one round (run under gpurun): launch list of one cfg2
# factorization + one `ncu --set full` capture per top kernel family, and the
# column-ring Jacobi kernel on cfg1 (l = 60).
# usage: bash tools/profile_round.sh r05   -> gpurun_out/<tag>_*.{csv,ncu-rep}
# (FFB_JACOBI_NOFUSE: ncu cannot replay the fused cooperative+cluster Jacobi
#  launch faithfully; FFB_GRAPHS=0: one node per launch in the list)
tag=${1:-r05}
export FFB_JACOBI_NOFUSE=1 FFB_GRAPHS=0
one="python tools/one_factorization.py --workload cfg2 --warmup 1"
one1="python tools/one_factorization.py --workload cfg1 --warmup 1"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches_cfg2.csv $one > gpurun_out/${tag}_ncu_list.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches_cfg1.csv $one1 > gpurun_out/${tag}_ncu_list1.log 2>&1
full="ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -c 1"
$full -k "regex:gemm_f64_kernel<\(int\)64, \(int\)144" -o gpurun_out/${tag}_k13 $one > gpurun_out/${tag}_ncu_k13.log 2>&1
$full -k "regex:gemm_f64_kernel<\(int\)80, \(int\)64, \(int\)16, \(int\)40, \(int\)32, \(bool\)1" -o gpurun_out/${tag}_sketch $one > gpurun_out/${tag}_ncu_sketch.log 2>&1
$full -k "regex:jacobi_kernel" -o gpurun_out/${tag}_jacobi $one > gpurun_out/${tag}_ncu_jacobi.log 2>&1
$full -k "regex:panel_qr_kernel" -o gpurun_out/${tag}_panel $one > gpurun_out/${tag}_ncu_panel.log 2>&1
$full -k "regex:pivots_kernel" -o gpurun_out/${tag}_pivots $one > gpurun_out/${tag}_ncu_pivots.log 2>&1
$full -k "regex:jacobi_ring_kernel" -o gpurun_out/${tag}_ring $one1 > gpurun_out/${tag}_ncu_ring.log 2>&1
# summaries made on the box; the two GEMM reports (40 MB each with sources) stay there
python tools/ncu_summary.py gpurun_out/${tag}_k13.ncu-rep gpurun_out/${tag}_sketch.ncu-rep gpurun_out/${tag}_jacobi.ncu-rep \
    gpurun_out/${tag}_panel.ncu-rep gpurun_out/${tag}_pivots.ncu-rep gpurun_out/${tag}_ring.ncu-rep > gpurun_out/${tag}_ncu_full_summary.txt 2>&1
python tools/ncu_traffic.py gpurun_out/${tag}_traffic.json gpurun_out/${tag}_k13.ncu-rep gpurun_out/${tag}_sketch.ncu-rep gpurun_out/${tag}_jacobi.ncu-rep \
    gpurun_out/${tag}_panel.ncu-rep gpurun_out/${tag}_pivots.ncu-rep gpurun_out/${tag}_ring.ncu-rep --pick "gemm_f64_kernel=64, 144" > gpurun_out/${tag}_traffic.log 2>&1
for k in jacobi panel pivots ring; do
  python tools/ncu_lines_cuda.py gpurun_out/${tag}_$k.ncu-rep 0 25 > gpurun_out/${tag}_hot_$k.txt 2>&1
done
rm -f gpurun_out/${tag}_k13.ncu-rep gpurun_out/${tag}_sketch.ncu-rep
ls -la gpurun_out/${tag}_*
