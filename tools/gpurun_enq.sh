timeout 300 python tools/enqueue_probe.py 8 2>&1 | tail -1
PF_NO_PDL=1 timeout 300 python tools/enqueue_probe.py 8 2>&1 | tail -1
PF_LANES=1 timeout 300 python tools/enqueue_probe.py 8 2>&1 | tail -1
