#!/bin/bash
# GPU-box helper: key ncu metrics of the block kernels (K=fwd|bwd) for each library given
# (""= in-tree): time, cycles, tensor pipe, MUFU (xu), shared memory and L2 throughput.
LIBS=("$@"); [ ${#LIBS[@]} -eq 0 ] && LIBS=("")
K=${K:-fwd}
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.avg.per_cycle_active
for v in "${LIBS[@]}"; do
  echo "== ${v:-main} ${WL:-gpt} $K"
  WF_LIB_PATH=$v timeout -s KILL 300 ncu --metrics $M --clock-control none -k regex:wf_block_$K -s 1 -c 1 --csv \
    python tools/kprof.py > gpurun_out/ncu_raw.txt 2>&1
  python tools/ncu_csv.py < gpurun_out/ncu_raw.txt || tail -5 gpurun_out/ncu_raw.txt
done
