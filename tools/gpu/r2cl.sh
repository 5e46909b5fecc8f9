mkdir -p gpurun_out
rm -f gpurun_out/parity_scale.jsonl
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
cp gpurun_out/parity_scale.jsonl gpurun_out/r2cl_parity_scale.jsonl 2>/dev/null
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2cl_bench.json 2> gpurun_out/r2cl_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2cl_ref.json 2>&1; echo ref rc=$?
timeout 1500 python tools/sweep.py --set all --out gpurun_out/r2cl_sweep.json 2>&1 | cut -c1-120
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2cl_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2cl_ncu.log 2>&1; echo ncu rc=$?
