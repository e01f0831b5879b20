timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scratch/ktime.py c2 200
KT_GRAPH=1 python scratch/ktime.py c2 200
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"topk|maxsim|plan" -s 30 -c 6 --csv python scratch/ktime.py c2 20 2>/dev/null | grep -E "topk|maxsim|plan" | awk -F, '{gsub(/"/,""); print $5, $NF}'
