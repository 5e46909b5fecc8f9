for a in "1 3 1 9 21 20" "1 3 2 8 32 32" "3 3 2 24 67 64" "1 3 1 9 16 16"; do timeout 60 python tools/gpu/probe_direct.py $a 2>&1 | tail -4; done
