# small-kernel select loops unrolled x8 vs not (tools/ab/selnu): small tests, C1 timeline + synchronous latency
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_small_gpu.py tests/test_sharded_gpu.py -q -x > gpurun_out/pytest_sel3.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_sel3.log
cp paper_2312_05417_b200/lib/libespn_gpu.so /tmp/prod_libespn_gpu.so
for r in 1 2; do
for v in unroll plain; do
  if [ $v = unroll ]; then cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so; else cp tools/ab/selnu/libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so; fi
  echo "$v $(timeout 300 python tools/small_timeline.py 1 2>&1 | tail -1)"
  echo "$v $(timeout 120 ./tools/c1_latency 3)"
done
done
cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so
