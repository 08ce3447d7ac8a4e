set -e
timeout 300 python tools/prof_solver.py > gpurun_out/prof_plain.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sweep_own" -s 31 -c 1 -o gpurun_out/prof_cur -f python tools/prof_solver.py > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
