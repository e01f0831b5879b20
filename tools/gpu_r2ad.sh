L=paper_2312_05417_b200/lib/libespn_gpu.so
for v in base orignow noprof2 late2 base orignow noprof2 late2; do cp tools/ab/libespn_gpu_$v.so $L; printf "%s " $v; timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
cp tools/ab/libespn_gpu_orignow.so $L
