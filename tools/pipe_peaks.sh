#!/bin/bash
# Measured pipe throughputs (tools/pipe_peaks.cu) -> gpurun_out/pipe_peaks.json (GPU box).
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/kl_pipe_peaks tools/pipe_peaks.cu && /tmp/kl_pipe_peaks > gpurun_out/pipe_peaks.json
cat gpurun_out/pipe_peaks.json
