timeout 300 python tools/waves_twice.py C4 15 2>&1 | tail -3
SPAND_RRQR_CLUSTER=8 timeout 300 python tools/waves_twice.py C4 15 2>&1 | tail -3
