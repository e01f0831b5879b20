# one full ncu capture of the MaxSim kernel in the C2 bench (source-level), plus the launch list
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 6 -c 1 -o gpurun_out/prof_maxsim -f python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|topk|plan|finalize|gather|merge" -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu=$?
