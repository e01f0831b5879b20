# launch list of the bench command + one full capture of the MaxSim kernel
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|topk|plan|gather|merge" -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 5 -c 1 -o gpurun_out/prof_maxsim -f python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
