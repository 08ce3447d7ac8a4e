# launch list + DRAM traffic of every kernel of one config-5 solve (bench defaults,
# sweep-by-sweep launches so ncu sees each kernel; graphs with conditional nodes are not profilable)
set -e
timeout 300 python tools/prof_solver.py > gpurun_out/prof_plain.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/traffic.csv python tools/prof_solver.py > gpurun_out/ncu_traffic.log 2>&1
echo done
