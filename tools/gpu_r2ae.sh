L=paper_2312_05417_b200/lib/libespn_gpu.so
for v in cur d1 late d1late cur d1 late d1late; do cp tools/ab/libespn_gpu_$v.so $L; printf "%s " $v; timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
cp tools/ab/libespn_gpu_cur.so $L
