for v in 0 4 8; do echo "L2AHEAD=$v"; RD_L2AHEAD=$v timeout 300 python tools/quick_time.py 2>&1 | grep -E "C3 float(64|32) thread"; done
