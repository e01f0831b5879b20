set -x
timeout 300 python -m pytest tests/test_server_gpu.py -x -q > gpurun_out/pytest_server.log 2>&1; echo server_tests=$?
tail -30 gpurun_out/pytest_server.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_d.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_d.log
