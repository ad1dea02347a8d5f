mkdir -p gpurun_out/tr_a gpurun_out/tr_b
MDD_LIB_PATH=$PWD/paper_2311_18783_b200/libmdd_x_nocompute.so MDD_SWEEP_TRACE=gpurun_out/tr_a timeout 600 python tools/ncu_c4.py sweeps c4 > gpurun_out/tr_a/run.log 2>&1
MDD_LIB_PATH=$PWD/paper_2311_18783_b200/libmdd_x_nocompute.so MDD_SWEEP_TRACE=gpurun_out/tr_b MDD_NOCOMPUTE=1 timeout 600 python tools/ncu_c4.py sweeps c4 > gpurun_out/tr_b/run.log 2>&1
for d in tr_a tr_b; do python tools/trace_report.py gpurun_out/$d/trace_local.bin > gpurun_out/$d/local.txt; python tools/trace_report.py gpurun_out/$d/trace_coarse.bin > gpurun_out/$d/coarse.txt; done
