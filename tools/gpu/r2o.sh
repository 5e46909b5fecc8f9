NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none -k regex:gather_rows -c 1 -o gpurun_out/r2o_g112 python tools/one_conv.py gather 128 56 232 225 112 > /dev/null 2>&1
$NCU --set full --clock-control none -k regex:gather_rows -c 1 -o gpurun_out/r2o_g496 python tools/one_conv.py gather 128 14 1024 1016 496 > /dev/null 2>&1
ls gpurun_out
