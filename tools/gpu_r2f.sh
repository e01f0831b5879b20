set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ivf_prefetch.py tests/test_cpp_api.py tests/test_server_gpu.py -x -q > gpurun_out/pytest_f.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_f.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo bench=$?
tail -3 gpurun_out/bench_f.err
