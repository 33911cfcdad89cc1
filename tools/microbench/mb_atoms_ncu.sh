#!/bin/bash
# ncu counters of the ATOMS pattern microbenchmark: shared-atomic wavefronts per instruction vs
# duration for each address pattern (round-2 study; profiles/r02_atoms_patterns_ncu.csv)
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_atoms_pattern mb_atoms_pattern.cu || exit 1
./mb_atoms_pattern > /dev/null || exit 1
ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__sass_inst_executed_op_shared_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum \
    --clock-control none -c 8 --csv --log-file "$1" ./mb_atoms_pattern > /dev/null
