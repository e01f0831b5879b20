set -x
ls /proc/driver/nvidia-fs 2>&1 | head -3; cat /proc/driver/nvidia-fs/stats 2>&1 | head -5; lsmod 2>/dev/null | grep -i nvidia_fs; ls /usr/local/cuda/gds/tools/gdscheck* 2>&1 | head -2; /usr/local/cuda/gds/tools/gdscheck -p 2>&1 | head -40 > gpurun_out/gdscheck.txt; df -hT /tmp /root 2>&1 | head -5; mount | grep -E " / | /tmp " | head
timeout 300 tests/cpp/refapi_test > gpurun_out/refapi_test.log 2>&1; echo refapi=$?; tail -5 gpurun_out/refapi_test.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_api.py tests/test_ivf_prefetch.py -x -q > gpurun_out/pytest_g.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_g.log
