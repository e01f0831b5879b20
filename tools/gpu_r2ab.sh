# MMA descriptor A/B (served C2 step) + quick parity
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05 or fp32 or c2 or c3 or fused" > gpurun_out/pytest_ab.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_ab.log
L=paper_2312_05417_b200/lib/libespn_gpu.so
for v in base desc base desc; do cp tools/ab/libespn_gpu_$v.so $L; printf "%s " $v; timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
cp tools/ab/libespn_gpu_desc.so $L
timeout 300 python tools/role_profile.py on 2>&1 | tail -18
