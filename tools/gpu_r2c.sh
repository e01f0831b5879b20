set -x
timeout 900 python -m pytest tests/test_sharded_gpu.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_c.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_c.log
timeout 900 python bench.py --gpus 2 --steps 50 --warmup 5 --preroll-s 0.5 --no-cpu-baseline > gpurun_out/bench_n2_replica.json 2> gpurun_out/bench_n2_replica.err; echo n2r=$?
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 3 --placement shard > gpurun_out/bench_n2_shard.json 2> gpurun_out/bench_n2_shard.err; echo n2s=$?
for f in gpurun_out/bench_n2_*.err; do tail -n 4 $f; done
