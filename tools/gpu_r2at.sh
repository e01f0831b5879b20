L=paper_2312_05417_b200/lib/libespn_gpu.so
for v in np16b cur2; do cp tools/ab/libespn_gpu_$v.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_server_gpu.py tests/test_fuzz_gpu.py -q -x -k "not small" > gpurun_out/pytest_at_$v.log 2>&1; echo pytest_$v=$?; tail -2 gpurun_out/pytest_at_$v.log; done
for v in cur np16b cur2 cur np16b cur2; do cp tools/ab/libespn_gpu_$v.so $L; printf "%s " $v; timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
cp tools/ab/libespn_gpu_cur.so $L
