# A/B: d=32 N=64 MMAs (NQC 64, 16 KB stages, 6 or 8 deep) vs production; parity of the variant
mkdir -p gpurun_out
VARIANTS="prod q64ns8 q64ns6" bash tools/gpu_r2be.sh
cp tools/ab/q64ns8/libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_server_gpu.py -x -q 2>&1 | tail -3
cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so
