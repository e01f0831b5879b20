# server-mode in-flight sweep (C2), C1 bench, sanitizers
for nl in 4 6; do
timeout 600 python bench.py --no-cpu-baseline --inflight $nl --steps 400 > gpurun_out/bench_i_nl$nl.json 2> gpurun_out/bench_i_nl$nl.err; echo nl$nl=$?
python -c "import json;r=json.load(open('gpurun_out/bench_i_nl$nl.json'));print($nl, r['value'], r['e2e']['value'], r['roofline']['frac'], r['clocks']['sm_mhz'], r['p50_batch_ms'])"
done
timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 200 --warmup 10 > gpurun_out/bench_i_c1.json 2> gpurun_out/bench_i_c1.err; echo c1=$?
cat gpurun_out/bench_i_c1.json | head -c 600; echo
SAN_TIMEOUT=700 bash tools/sanitize.sh
