# small kernel v2 (batched metadata, smem row staging; opt-in), gather v2, suite, sanitizers, probes
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests/test_small_gpu.py -x -q > gpurun_out/pytest_m_small.log 2>&1; echo small=$?; tail -3 gpurun_out/pytest_m_small.log
for k in 1 3; do timeout 120 ./tools/c1_latency $k; done > gpurun_out/c1_latency_m.txt 2>&1; cat gpurun_out/c1_latency_m.txt
timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 200 --warmup 10 > gpurun_out/bench_m_c1.json 2> gpurun_out/bench_m_c1.err; echo c1=$?
head -c 2600 gpurun_out/bench_m_c1.json | tail -c 1400; echo
compute-sanitizer --tool racecheck ./tools/racecheck_probe > gpurun_out/racecheck_probe_m.txt 2>&1; grep -v "^=========     at" gpurun_out/racecheck_probe_m.txt | head -30
for t in "tests/test_gpu_parity.py::test_tiered_store_matches_resident_and_oracle[simt]" "tests/test_gpu_parity.py::test_c1_shape_parity[simt]" "tests/test_gpu_parity.py::test_tiered_store_matches_resident_and_oracle[tcgen05]"; do
  timeout 600 compute-sanitizer --tool initcheck --print-limit 3 python -m pytest "$t" -x -q -p no:cacheprovider 2>&1 | grep -v "Host Frame\|^=========     at" | tail -25
done > gpurun_out/initcheck_m.txt 2>&1; cat gpurun_out/initcheck_m.txt | head -80
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_m.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_m.log
timeout 600 python bench.py > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; echo bench=$?; python -c "import json;r=json.load(open('gpurun_out/bench_m.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['gather_hbm_gbs'],r['clocks'])"
SAN_TIMEOUT=700 bash tools/sanitize.sh
