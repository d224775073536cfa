for M in 1 8; do timeout 300 python tools/enqueue_probe.py $M 2>&1 | tail -1; done
