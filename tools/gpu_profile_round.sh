set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:mdd:: --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu1 rc $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_sweep -s 5 -c 1 -o gpurun_out/prof_local python tools/diag_sweep.py c1 > gpurun_out/ncu_local.log 2>&1; echo ncu2 rc $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_sweep -s 30 -c 1 -o gpurun_out/prof_coarse python tools/diag_sweep.py c1 > gpurun_out/ncu_coarse.log 2>&1; echo ncu3 rc $?
