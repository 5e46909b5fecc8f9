timeout 1500 python tools/sweep.py --set all --out gpurun_out/r2f_sweep.json 2>&1 | tail -20
