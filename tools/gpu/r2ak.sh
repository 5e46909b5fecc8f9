for f in 0 64 4 16 20 84; do echo "flags $f: $(UB_DEBUG_FLAGS=$f python tools/bench_stem.py 2>&1 | head -1)"; done
echo "tma store: $(UB_SP_TMA_STORE=1 python tools/bench_stem.py 2>&1 | head -1)"
echo "sleep 100: $(UB_SP_SLEEP=100 python tools/bench_stem.py 2>&1 | head -1)"
python tools/bench_stem.py 2>&1 | tail -4
