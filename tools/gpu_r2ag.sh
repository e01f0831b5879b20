L=paper_2312_05417_b200/lib/libespn_gpu.so
for v in cur g4 g6 cur g4 g6; do cp tools/ab/libespn_gpu_$v.so $L; timeout 600 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ag_$v.json 2>/dev/null; python -c "import json;r=json.load(open('gpurun_out/bench_ag_$v.json'));print('$v', r['gather_hbm_gbs'], r['value'], r['clocks']['sm_mhz'])"; done
cp tools/ab/libespn_gpu_cur.so $L
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|plan|finalize|wait|gather" -c 120 --csv --log-file gpurun_out/launches_v2.csv python bench.py --steps 20 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_launch_v2.log 2>&1; echo ncu=$?
