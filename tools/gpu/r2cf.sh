mkdir -p gpurun_out
rm -f gpurun_out/parity_scale.jsonl
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
cp gpurun_out/parity_scale.jsonl gpurun_out/r2cf_parity_scale.jsonl 2>/dev/null
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2cf_bench.json 2> gpurun_out/r2cf_bench.err; echo bench rc=$?
timeout 1500 python tools/sweep.py --set all --out gpurun_out/r2cf_sweep.json 2>&1 | cut -c1-200
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
