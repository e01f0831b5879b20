# small kernel (k-way merge), all-lane arrives in the MaxSim kernel: suite, latency, C1/C2 bench, sanitizers
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests/test_small_gpu.py -x -q > gpurun_out/pytest_l_small.log 2>&1; echo small=$?; tail -3 gpurun_out/pytest_l_small.log
for k in 1 3 0; do timeout 120 ./tools/c1_latency $k; done > gpurun_out/c1_latency_l.txt 2>&1; cat gpurun_out/c1_latency_l.txt
timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 200 --warmup 10 > gpurun_out/bench_l_c1.json 2> gpurun_out/bench_l_c1.err; echo c1=$?
head -c 2500 gpurun_out/bench_l_c1.json; echo
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_l.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_l.log
timeout 600 python bench.py > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; echo bench=$?; head -c 3000 gpurun_out/bench_l.json; echo
SAN_TIMEOUT=700 bash tools/sanitize.sh
