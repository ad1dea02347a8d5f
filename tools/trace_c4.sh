#!/bin/bash
# per-phase sweep timelines of the c4 local and coarse sweeps (B200)
mkdir -p gpurun_out/trace_c4
MDD_SWEEP_TRACE=gpurun_out/trace_c4 MDD_PLAN_STATS=1 python tools/ncu_c4.py sweeps c4 > gpurun_out/trace_c4/run.log 2>&1
python tools/trace_report.py gpurun_out/trace_c4/trace_local.bin > gpurun_out/trace_c4/local.txt
python tools/trace_report.py gpurun_out/trace_c4/trace_coarse.bin > gpurun_out/trace_c4/coarse.txt
