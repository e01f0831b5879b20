# final-kernel ncu full capture (non-persistent launch) + launch list
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 5 -c 1 -o gpurun_out/prof_maxsim_final -f python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_full_final.log 2>&1; echo ncufull=$?
ncu -i gpurun_out/prof_maxsim_final.ncu-rep --page raw --csv > gpurun_out/maxsim_raw_final.csv 2>&1; echo raw=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|plan|finalize|wait|gather" -c 120 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 20 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_launch_final.log 2>&1; echo ncu=$?
