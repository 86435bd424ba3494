import sys
sys.path.insert(0, '.')
from paper_2406_17284_b200 import ltl
pre = ltl.ltl_presets()
with ltl.DeviceTorus(rows=32768, cols=32768) as t:
    for r in (1, 2):
        name, rule, dens = pre[r - 1]
        t.init_random(dens, 1)
        t.run(rule, 1, engine="pack")
