#!/bin/bash
# Round-end measurement on one B200: the bench line, the launch list of the hot
# path (profiler range of tools/ncu_c4.py), and ncu --set full of both sweeps and
# of the other solve kernels.  Outputs under gpurun_out/prof/.
set -x
O=gpurun_out/prof
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc $?
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --kernel-name-base demangled --csv --log-file $O/launches.csv python tools/ncu_c4.py solve > $O/ncu_launches.log 2>&1
echo launches rc $?
python tools/launch_shares_all.py $O/launches.csv > $O/launch_shares.txt 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k regex:k_sweep -c 2 -o $O/sweeps python tools/ncu_c4.py sweeps > $O/ncu_sweeps.log 2>&1
echo sweeps rc $?
if [ -z "$SKIP_SOLVE_KERNELS" ]; then   # (unchanged kernels need no re-capture)
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k regex:"k_spmv|k_geneo|k_z_apply|k_update|k_dot" -c 12 -o $O/solve_kernels \
  python tools/ncu_c4.py solve > $O/ncu_solve_kernels.log 2>&1
echo solve kernels rc $?
fi
python tools/ncu_summary.py $O/sweeps.ncu-rep "c4 sweeps (local, coarse)" "tools/ncu_c4.py sweeps" > $O/ncu_sweeps.json
[ -z "$SKIP_SOLVE_KERNELS" ] && python tools/ncu_summary.py $O/solve_kernels.ncu-rep "c4 solve kernels" "tools/ncu_c4.py solve" > $O/ncu_solve_kernels.json
ls -la $O
