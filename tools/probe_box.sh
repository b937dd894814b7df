#!/bin/bash
# One-off box probe: host cores/RAM, GPU, FP64 pipe peaks.
mkdir -p gpurun_out
{
nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; free -g; nvidia-smi; 
./tools/fp64_peak
} > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt | tail -60
