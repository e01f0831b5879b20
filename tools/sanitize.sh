# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over the
# library's kernels on small parity cases: C2-shaped d=32 (fused top-k), d=128
# (REPA, the C3 shard kernel), fp32-query split, tiered + prefetch, separate
# top-k, gather, persistent server.  Logs -> gpurun_out/sanitize_*.log
K='--kernel-name regex=rerank_small|relocate|synth|tile_jobs|maxsim|plan_|finalize|stage|topk|gather|merge|tile_rows|hint|count_|wait_'
T="tests/test_gpu_parity.py::test_c1_shape_parity tests/test_gpu_parity.py::test_tcgen05_dims_dtypes tests/test_gpu_parity.py::test_fp32_query_parity_dims tests/test_gpu_parity.py::test_tiered_store_matches_resident_and_oracle tests/test_gpu_parity.py::test_prefetch_on_off_identical_and_hit_rate tests/test_gpu_parity.py::test_fused_topk_ragged_and_empty_queries tests/test_gpu_parity.py::test_fused_topk_matches_separate tests/test_gpu_parity.py::test_gather_bitexact tests/test_gpu_parity.py::test_merge_topk tests/test_server_gpu.py::test_served_equals_unserved_and_oracle tests/test_small_gpu.py::test_c1_shape_bitexact tests/test_small_gpu.py::test_errors_and_recovery"
# initcheck without a kernel filter: a filtered run does not see the writes of
# the kernels it skips, so memory they initialise reads as uninitialised
for tool in memcheck racecheck synccheck initcheck; do
  KF="$K"; [ $tool = initcheck ] && KF=""
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool $KF --print-limit 50 --log-file gpurun_out/sanitize_$tool.log \
    python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/sanitize_${tool}_pytest.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log; tail -2 gpurun_out/sanitize_${tool}_pytest.log
done
