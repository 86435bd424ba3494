#!/bin/bash
# A/B: CUDA-core engines' CTAs per SM (dynamic SMEM floor / padding), 32768^2.
set -u
cat > /tmp/pk.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2406_17284_b200 import ltl
n = 32768
eng = sys.argv[1]
with ltl.DeviceTorus(n=n) as t:
    out = []
    for text, d in (("R1,C2,M0,S2..3,B3..3,NM", .07), ("R2,C2,M0,S7..12,B8..11,NM", .15), ("R3,C2,M0,S15..23,B14..17,NM", .25), ("R8,C2,M0,S163..223,B74..252,NM", .23), ("R16,C2,M0,S170..296,B170..300,NM", .26)):
        t.init_random(d, 1)
        tot, _ = t.time(text, 10, 3, engine=eng)
        out.append("r%s %.1f us" % (text[1:text.index(',')], tot / 10 * 1e3))
print(eng, os.environ.get("LTL_BASE_PAD_SMEM", os.environ.get("LTL_PACK_MIN_SMEM", "default")), " | ".join(out), flush=True)
PY
timeout 300 python /tmp/pk.py pack
for m in 0 2000 10000 18000 30000; do LTL_BASE_PAD_SMEM=$m timeout 300 python /tmp/pk.py base; done
