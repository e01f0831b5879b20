# all bench configs on one GPU (C3/C5 as the per-GPU share of the 8-way sharding)
set -x
timeout 600 python bench.py --no-cpu-baseline --config c3 --emulate-shards 8 --steps 50 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 900 python bench.py --no-cpu-baseline --config c5 --emulate-shards 8 --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
timeout 600 python bench.py --no-cpu-baseline --config c4 --steps 100 --warmup 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 100 --warmup 10 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo c1=$?
