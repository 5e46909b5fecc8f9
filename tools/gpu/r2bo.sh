mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_scale.py -m gpu -q -x -k "mobilenet or efficientnet" 2>&1 | tail -3
cp gpurun_out/parity_scale.jsonl gpurun_out/r2bo_parity_scale.jsonl 2>/dev/null
timeout 1200 python tools/sweep.py --set config5 --out gpurun_out/r2bo_sweep_config5.json 2>&1 | cut -c1-330
timeout 900 python tools/sweep.py --set mobilenet --out gpurun_out/r2bo_sweep_mobilenet.json 2>&1 | cut -c1-250
