#!/bin/bash
# ncu counters of every d = 1 spreading formulation of mb_spread2.cu (verdict r01 #2: "profiles must
# hold the ncu counters of every variant tried"): duration, warp-instructions, shared-atomic
# instructions and wavefronts, l1tex and issue utilisation per kernel (profiles/r02_spread_variants_ncu.csv)
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mb_spread2 mb_spread2.cu || exit 1
./mb_spread2 > /dev/null || exit 1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__sass_inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum \
    -k regex:"k_base|k_lean|k_quad|k_pair|math" --clock-control none -c 60 --csv --log-file "$1" ./mb_spread2 > /dev/null
