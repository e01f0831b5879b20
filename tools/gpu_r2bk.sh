# small-batch kernel: last-CTA merge by threshold select vs the two-level k-way merge (ESPN_SMALL_SELECT=0 in tools/ab/sel0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_small_gpu.py tests/test_fuzz_gpu.py tests/test_sharded_gpu.py -q -x > gpurun_out/pytest_sel.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_sel.log
cp paper_2312_05417_b200/lib/libespn_gpu.so /tmp/prod_libespn_gpu.so
for r in 1 2; do
for v in select kway; do
  if [ $v = select ]; then cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so; else cp tools/ab/sel0/libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so; fi
  timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 200 --warmup 10 > gpurun_out/bench_sel_c1_$v.json 2> gpurun_out/bench_sel_c1_$v.err
  python -c "import json;r=json.load(open('gpurun_out/bench_sel_c1_$v.json'));print('$v',r['value'],r['e2e']['value'],r['p50_batch_ms'],r['roofline']['kernel_ms'],r['roofline']['exclusive']['kernel_ms'],r['clocks']['sm_mhz'],r['config'].get('kernel'),r.get('check'))"
  timeout 300 python tools/small_timeline.py 1 2>&1 | tail -1
done
done
cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so
