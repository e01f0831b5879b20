L=paper_2312_05417_b200/lib/libespn_gpu.so
cp tools/ab/libespn_gpu_lw64.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_server_gpu.py -q -x -k "not small" > gpurun_out/pytest_av.log 2>&1; echo pytest_lw64=$?; tail -2 gpurun_out/pytest_av.log
for v in cur lw64 cur lw64; do cp tools/ab/libespn_gpu_$v.so $L; printf "%s " $v; timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
cp tools/ab/libespn_gpu_cur.so $L
