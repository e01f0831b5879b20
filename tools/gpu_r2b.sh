set -x
timeout 900 python -m pytest tests/test_sharded_gpu.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_b.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_b.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo n1=$?
timeout 900 python bench.py --gpus 2 --steps 50 --warmup 5 --preroll-s 0.5 > gpurun_out/bench_n2_replica.json 2> gpurun_out/bench_n2_replica.err; echo n2r=$?
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 3 --placement shard > gpurun_out/bench_n2_shard.json 2> gpurun_out/bench_n2_shard.err; echo n2s=$?
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 3 --placement replica-split > gpurun_out/bench_n2_rsplit.json 2> gpurun_out/bench_n2_rsplit.err; echo n2rs=$?
tail -3 gpurun_out/*.err
