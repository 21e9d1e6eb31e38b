timeout 600 python tools/init_timing.py cfg2 2>&1 | tail -30
