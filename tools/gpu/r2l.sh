timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/bench_gather.py 2>&1 | tail -6
timeout 300 python tools/op_times.py densenet121_s50 128 2>&1 | head -1
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 2>&1 | head -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo rc=$?; tail -3 gpurun_out/r2l_bench.err
