# small kernel: L2 prefetch of candidate rows (tools/ab/l2pf, ESPN_SMALL_L2PF=1) vs production; C1 timeline + synchronous latency; parity of the variant
mkdir -p gpurun_out
cp paper_2312_05417_b200/lib/libespn_gpu.so /tmp/prod_libespn_gpu.so
for r in 1 2; do
for v in prod l2pf; do
  if [ $v = prod ]; then cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so; else cp tools/ab/l2pf/libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so; fi
  echo "$v $(timeout 300 python tools/small_timeline.py 1 2>&1 | tail -1)"
  echo "$v $(timeout 120 ./tools/c1_latency 3)"
done
done
cp tools/ab/l2pf/libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so
timeout 600 python -m pytest tests/test_small_gpu.py -q -x 2>&1 | tail -1
cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so
