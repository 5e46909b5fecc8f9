rm -f gpurun_out/parity_scale.jsonl
timeout 1500 python -m pytest tests/test_parity_scale.py -m gpu -q -k "mobilenet or efficientnet or resnet50_s50-reorder" 2>&1 | tail -3
cat gpurun_out/parity_scale.jsonl
