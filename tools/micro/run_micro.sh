#!/bin/bash
# One-off probe: fp64 pipe ceilings, cuBLAS DGEMM comparator, host facts.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/micro_smi.txt 2>&1
lscpu > gpurun_out/micro_lscpu.txt 2>&1
free -g > gpurun_out/micro_free.txt 2>&1
nproc >> gpurun_out/micro_free.txt
python -c "import os; print(len(os.sched_getaffinity(0)))" >> gpurun_out/micro_free.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/micro_clocks.csv &
CLK=$!
timeout 120 ./tools/micro/fp64_peak > gpurun_out/micro_fp64.jsonl 2>&1
timeout 300 python tools/micro/torch_dgemm.py >> gpurun_out/micro_fp64.jsonl 2>&1
kill $CLK
