#!/bin/bash
# count distinct Jacobi trajectories / R factors of a repeated fuzz case (expect 1 / 1)
C=${1:-3}; R=${2:-40}
FFB_JACOBI_PROF=1 timeout 300 python tools/probe/jac_rep.py $C $R > /tmp/o.txt 2> /tmp/e.txt
echo "== case $C: distinct offmax: $(grep offmax /tmp/e.txt | sort -u | wc -l)  distinct (ds,dR): $(awk '{print $(NF-2), $NF}' /tmp/o.txt | sort -u | wc -l) errs: $(grep -c ERR /tmp/o.txt)"
