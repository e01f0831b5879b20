# small-batch single-launch kernel: parity, latency floor, C1 bench; racecheck model probe; DRAM traffic probe
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests/test_small_gpu.py -x -q > gpurun_out/pytest_k_small.log 2>&1; echo small=$?; tail -15 gpurun_out/pytest_k_small.log
./tools/c1_floor > gpurun_out/c1_floor.txt 2>&1; cat gpurun_out/c1_floor.txt
for k in 1 3 0; do timeout 120 ./tools/c1_latency $k; done > gpurun_out/c1_latency_k.txt 2>&1; cat gpurun_out/c1_latency_k.txt
compute-sanitizer --tool racecheck ./tools/racecheck_probe > gpurun_out/racecheck_probe.txt 2>&1; cat gpurun_out/racecheck_probe.txt | grep -v "^=========     at" | head -60
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --csv ./tools/traffic_probe > gpurun_out/traffic_probe.csv 2>&1; echo ncu=$?
grep -v "^==PROF==" gpurun_out/traffic_probe.csv | head -5
for kk in auto tcgen05; do
timeout 300 python bench.py --no-cpu-baseline --config c1 --kernel $kk --steps 200 --warmup 10 > gpurun_out/bench_k_c1_$kk.json 2> gpurun_out/bench_k_c1_$kk.err; echo c1_$kk=$?
head -c 1500 gpurun_out/bench_k_c1_$kk.json; echo; tail -2 gpurun_out/bench_k_c1_$kk.err
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_k.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_k.log
