# ncu full-set capture of the small-batch kernel with the threshold-select merge (C1)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rerank_small -s 5 -c 1 -o gpurun_out/prof_small_sel -f python bench.py --config c1 --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline > gpurun_out/ncu_small_sel.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_small_sel.ncu-rep --page details --csv > gpurun_out/small_sel_details.csv 2>&1; echo details=$?
