set -x
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_e.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_e.log
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|plan|finalize|gather|wait" -c 80 --csv --log-file gpurun_out/launches_r2_c2.csv python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 5 -c 1 -o gpurun_out/prof_maxsim_r2 python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
