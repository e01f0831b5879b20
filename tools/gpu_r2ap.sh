# final code verification + inflight sweep for the default bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_ap.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_ap.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for nl in 3 4 3 4; do timeout 600 python bench.py --no-cpu-baseline --inflight $nl --steps 400 > gpurun_out/bench_ap_$nl.json 2>/dev/null; python -c "import json;r=json.load(open('gpurun_out/bench_ap_$nl.json'));print($nl, r['value'],r['e2e']['value'],r['roofline']['frac'],r['clocks']['sm_mhz'])"; done
