"""Developer parity check: engine sweep vs the reference oracle on small cases."""
import json, sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from parity_util import parity_cases, diff_json
from paper_2506_04203_b200 import engine as eng
from oracle import refpy

E = eng.Engine(0)
ok = True
for name, t, cfg, N in parity_cases():
    t0 = time.time(); ref = refpy.sweep(t, cfg, N); tr = time.time() - t0
    for prune in (1, 0):
        E.set_option("prune", prune)
        t0 = time.time()
        try:
            got = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
        except Exception as ex:
            print(name, "ENGINE ERROR", ex); ok = False; continue
        tg = time.time() - t0
        d = diff_json(got, ref["result"])
        print(f"{name} prune={prune}: ref {tr:.2f}s gpu {tg:.3f}s evals={len(got['evaluations'])} diffs={len(d)}")
        for x in d[:10]: print("   ", x)
        print("   stats", {k: v for k, v in E.last_stats.items() if v})
        ok &= not d
print("ALL OK" if ok else "MISMATCH")
