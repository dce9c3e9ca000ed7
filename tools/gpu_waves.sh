#!/bin/bash
# Launch list with grid sizes, occupancy limits and waves per SM of the C4 setup kernels
# (cold_setup_probe c4: permutations, K4, seg layout three times) and one bench step.
mkdir -p gpurun_out
M=gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__waves_per_multiprocessor,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__occupancy_limit_warps,launch__registers_per_thread
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/waves_c4.csv python tools/cold_setup_probe.py c4 > gpurun_out/waves_c4.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/waves_c3.csv python tools/cold_setup_probe.py c3 > gpurun_out/waves_c3.log 2>&1
