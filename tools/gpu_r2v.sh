# round-2 final: every config on one GPU (C3/C5 as the per-GPU share of the 8-way sharding), C1 both kernels,
# the server-mode launch list, ncu full captures of the gather copy and small-batch kernels
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --config c3 --emulate-shards 8 --steps 50 --warmup 5 > gpurun_out/bench_v_c3.json 2> gpurun_out/bench_v_c3.err; echo c3=$?
timeout 900 python bench.py --no-cpu-baseline --config c5 --emulate-shards 8 --steps 20 --warmup 3 > gpurun_out/bench_v_c5.json 2> gpurun_out/bench_v_c5.err; echo c5=$?
timeout 600 python bench.py --no-cpu-baseline --config c4 --steps 100 --warmup 10 > gpurun_out/bench_v_c4.json 2> gpurun_out/bench_v_c4.err; echo c4=$?
timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 200 --warmup 10 > gpurun_out/bench_v_c1.json 2> gpurun_out/bench_v_c1.err; echo c1=$?
timeout 300 python bench.py --no-cpu-baseline --config c1 --kernel tcgen05 --steps 200 --warmup 10 > gpurun_out/bench_v_c1_tc.json 2> gpurun_out/bench_v_c1_tc.err; echo c1tc=$?
for f in c3 c5 c4 c1 c1_tc; do python -c "import json;r=json.load(open('gpurun_out/bench_v_$f.json'));print('$f', r['value'], r.get('e2e',{}).get('value'), r['roofline']['frac'] if 'roofline' in r else None, r['clocks'])" 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|plan|finalize|wait|gather|small" -c 120 --csv --log-file gpurun_out/launches_v.csv python bench.py --steps 20 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_launch_v.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_copy -s 3 -c 1 -o gpurun_out/prof_gather -f python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_gather.log 2>&1; echo ncugather=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rerank_small -s 5 -c 1 -o gpurun_out/prof_small -f python bench.py --config c1 --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_small.log 2>&1; echo ncusmall=$?
