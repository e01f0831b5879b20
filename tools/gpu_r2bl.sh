# threshold-select merge of the small-batch kernel: full small suite (incl. the k = 32 select / fallback test), fuzz, sharded; sanitizers on the small kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_small_gpu.py tests/test_fuzz_gpu.py tests/test_sharded_gpu.py -q -x > gpurun_out/pytest_sel2.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_sel2.log
T="tests/test_small_gpu.py::test_c1_shape_bitexact tests/test_small_gpu.py::test_last_cta_merge_select_and_fallback tests/test_small_gpu.py::test_errors_and_recovery tests/test_small_gpu.py::test_longest_lists_and_max_batch"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name regex=rerank_small --print-limit 50 --log-file gpurun_out/sanitize_small_$tool.log \
    python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/sanitize_small_${tool}_pytest.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_small_$tool.log; tail -1 gpurun_out/sanitize_small_${tool}_pytest.log
done
timeout 300 python bench.py --config c1 > gpurun_out/bench_r2_v12_c1.json 2> gpurun_out/bench_r2_v12_c1.err; echo c1=$?
python -c "import json;r=json.load(open('gpurun_out/bench_r2_v12_c1.json'));print(r['value'],r['e2e']['value'],r['p50_batch_ms'],r['roofline']['exclusive']['kernel_ms'],r['clocks'])"
