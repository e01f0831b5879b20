set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|topk|gather" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 5 -c 2 -o gpurun_out/prof_maxsim python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_copy -s 3 -c 1 -o gpurun_out/prof_gather python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_gather.log 2>&1; echo ncu3=$?
