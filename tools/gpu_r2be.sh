# A/B of d=32 work-unit geometry (UNITMAX x NU x NS), served C2 step, eager loop (tools/server_knobs.py)
# variants prebuilt in tools/ab/<name>/libespn_gpu.so by nvcc with ESPN_D32_* defines
mkdir -p gpurun_out
cp paper_2312_05417_b200/lib/libespn_gpu.so /tmp/prod_libespn_gpu.so
for r in 1 2 3; do
  for v in ${VARIANTS:-prod u128ns3 u96ns3 u160nu2 u192nu2ns3}; do
    if [ $v = prod ]; then cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so; else cp tools/ab/$v/libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so; fi
    echo "$v $(timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1)"
  done
done
cp /tmp/prod_libespn_gpu.so paper_2312_05417_b200/lib/libespn_gpu.so
