timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "gather or eltwise or dwconv or linear or avgpool or direct or permute or production" > gpurun_out/r2s_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -5 gpurun_out/r2s_memcheck.log
