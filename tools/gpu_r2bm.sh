# final tree after the small-kernel select: full GPU suite, smoke, batch-1 synchronous latency
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final2.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_final2.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
for k in 3 1; do timeout 120 ./tools/c1_latency $k; done
