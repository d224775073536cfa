for M in 8; do timeout 300 python tools/enqueue_probe.py $M 2>&1 | tail -1; done
which perf 2>/dev/null; ls /usr/bin/*perf* 2>/dev/null | head -3
