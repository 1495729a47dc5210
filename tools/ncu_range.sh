#!/bin/bash
# Aggregate ncu counters over one whole bench step (application-range replay), Kernelet vs the
# sequential baseline.  Outputs gpurun_out/range_{kernelet,sequential}.csv.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg
mkdir -p gpurun_out
for m in kernelet sequential; do
  timeout 1200 ncu --replay-mode app-range --clock-control none --metrics $M --csv \
    python tools/range_target.py $m > gpurun_out/range_$m.csv 2> gpurun_out/range_$m.err
  echo "$m exit $?"; grep -E '^"' gpurun_out/range_$m.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tr -d '"' | tail -14
done
