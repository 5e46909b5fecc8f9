timeout 600 python tools/sweep.py --set densenet 2>&1 | tail -1 | cut -c1-600
