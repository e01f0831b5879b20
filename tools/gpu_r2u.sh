# which path bounds the persistent server (ESPN_DEBUG knobs; invalid rankings by design)
for k in 0 4 1 2 3 32 0; do timeout 300 python tools/server_knobs.py $k on 2>&1 | tail -1; done
for k in 0 4 1; do timeout 300 python tools/server_knobs.py $k off 2>&1 | tail -1; done
