python tools/bench_variants.py 256 112 112 24 0 12 22 3 1 0 128 8 9 10 40 41 42
python tools/bench_variants.py 256 56 56 48 0 24 96 3 1 0 128 8 9 10 40 41 42
python tools/bench_variants.py 256 112 112 24 0 12 48 3 2 0 128 8 9 10 40 41 42
python tools/bench_variants.py 256 56 56 64 0 64 32 3 1 0 128 8 9 10
