#!/bin/bash
# Local-memory (spill) traffic and time of the frame kernel: in-tree lib and every lib_v* variant.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-extras --headstart-us 0"
M=l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 300 $CMD > gpurun_out/plain.log 2>&1 || exit 1
for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 600 ncu --metrics $M --clock-control none -k regex:frame_kernel -s 2 -c 1 --csv $CMD > gpurun_out/spill_$(basename $v).csv 2>gpurun_out/spill_$(basename $v).err; echo $v=$?
done
