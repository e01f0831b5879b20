# ncu full capture (source-level stall sampling) of the C2 MaxSim kernel, non-persistent launch
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 5 -c 1 -o gpurun_out/prof_maxsim_r2 -f python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_full_r2.log 2>&1; echo ncufull=$?
ncu -i gpurun_out/prof_maxsim_r2.ncu-rep --page source --csv --print-source sass > gpurun_out/maxsim_source_sass.csv 2>&1; echo src=$?
ncu -i gpurun_out/prof_maxsim_r2.ncu-rep --page source --csv --print-source cuda > gpurun_out/maxsim_source_cuda.csv 2>&1; echo srcc=$?
ncu -i gpurun_out/prof_maxsim_r2.ncu-rep --page raw --csv > gpurun_out/maxsim_raw_r2.csv 2>&1; echo raw=$?
ls -la gpurun_out/*.csv | tail -4
