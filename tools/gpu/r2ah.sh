rm -f gpurun_out/parity_scale.jsonl
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2h_ref.json 2>&1; echo ref rc=$?
timeout 1200 python tools/sweep.py --set all --out gpurun_out/r2h_sweep.json > /dev/null 2>&1; echo sweep rc=$?
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
