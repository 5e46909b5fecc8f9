NCU=/usr/local/cuda/bin/ncu
python tools/one_conv.py conv 256 112 112 12 22 3 1 24 0 && \
$NCU --set full --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/r2k_conv_small python tools/one_conv.py conv 256 112 112 12 22 3 1 24 0 > gpurun_out/r2k_ncu1.log 2>&1
python tools/one_conv.py gather 128 56 232 225 64 && \
$NCU --set full --clock-control none -k regex:gather_rows -c 1 -o gpurun_out/r2k_gather python tools/one_conv.py gather 128 56 232 225 64 > gpurun_out/r2k_ncu2.log 2>&1
ls -la gpurun_out/
