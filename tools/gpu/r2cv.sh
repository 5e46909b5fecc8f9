mkdir -p gpurun_out
rm -f gpurun_out/parity_scale.jsonl
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
cp gpurun_out/parity_scale.jsonl gpurun_out/r2cv_parity_scale.jsonl 2>/dev/null
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2cv_bench.json 2> gpurun_out/r2cv_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2cv_ref.json 2>&1; echo ref rc=$?
timeout 1500 python tools/sweep.py --set all --out gpurun_out/r2cv_sweep.json 2>&1 | cut -c1-120
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
