timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 > /tmp/o1.jsonl 2>&1
UB_SE_NOFUSEPOOL=1 timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 > /tmp/o2.jsonl 2>&1
head -1 /tmp/o1.jsonl | cut -c1-400; head -1 /tmp/o2.jsonl | cut -c1-400
python - <<'PY'
import json
for f in ('/tmp/o1.jsonl','/tmp/o2.jsonl'):
    L=[json.loads(l) for l in open(f) if l.startswith('{')][1:]
    dw=[r for r in L if r['kernel']=='dwconv_kernel']
    print(f, sorted([(r['op'][:16], r['us']) for r in dw], key=lambda t:-t[1])[:6])
PY
