# usage: bash tools/gpu_iter.sh [tests] [bench] [ncu] [ncufull]   (outputs in gpurun_out/)
set -x
for a in "$@"; do case $a in
tests) timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke.log;;
bench) timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err;;
ncu) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|topk|gather|merge" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu=$?;;
ncufull) timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 5 -c 1 -o gpurun_out/prof_maxsim -f python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?;;
esac; done
