for c in 32 64; do echo "cout $c"; UB_STEM_COUT=$c timeout 120 python tools/bench_stem.py | head -1; UB_SP_NOQUAD=1 UB_STEM_COUT=$c timeout 120 python tools/bench_stem.py | head -1; done
python - <<'PY'
import json
from paper_2307_08771_b200.configs import CONFIGS
PY
