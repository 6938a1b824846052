#!/bin/bash
# Bank-conflict attribution A/B: the same production kernels with and
# without their global loads / stores.  The variant library is built here with
#   python -m paper_1507_01391_b200.build -D DMM_NO_GLOBAL_IO
# (keys synthesised in registers, stores predicated off at run time) and selected through
# DMM_B200_LIB.  Run under gpurun on one B200, from the repo root.
set -e
VAR=paper_1507_01391_b200/_variants/libdmm_b200_dmm_no_global_io.so  # (python -m paper_1507_01391_b200.build -D DMM_NO_GLOBAL_IO)
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum,smsp__sass_inst_executed_op_global_ld.sum,smsp__sass_inst_executed_op_global_st.sum,gpu__time_duration.sum
mkdir -p gpurun_out
for CFG in cfg1 cfg3; do
  for V in prod noio; do
    if [ $V = noio ]; then export DMM_B200_LIB=$VAR; else unset DMM_B200_LIB; fi
    python tools/one_launch.py $CFG > gpurun_out/ab_plain_${CFG}_${V}.log 2>&1
    ncu --metrics $M --clock-control none -k regex:'k_general_sort|k_tile_sort' -c 1 --csv \
        python tools/one_launch.py $CFG > gpurun_out/ab_${CFG}_${V}.csv 2> gpurun_out/ab_${CFG}_${V}.err
  done
done
unset DMM_B200_LIB
echo "conflicts A/B done"
