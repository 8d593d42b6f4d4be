for d in 0 1 2 3; do echo "dbg=$d"; EWB_TC_DBG=$d python tools/tc_check.py c2 c3 c5 2>&1 | grep "tc=True"; done
