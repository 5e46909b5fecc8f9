set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo rc=$?
tail -5 gpurun_out/r2a_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2a_ref.json 2>&1; echo rc=$?
