import sys, json
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import scenarios as S, oracle
from paper_2510_09665_b200.api import Engine
C = oracle.C()
ref = json.loads(json.dumps(S._random_trace(oracle.RefEngine, C, 12, 7, decode=True, probe=True)))
got = json.loads(json.dumps(S._random_trace(Engine, C, 12, 7, decode=True, probe=True)))
for i, (x, y) in enumerate(zip(ref, got)):
    if i < 4: continue
    print("iter", i)
    print("   ref stores", [[s[3][:8] + f"({s[2]})" for s in p["store"]] for p in x["plans"]])
    print("   ref after batch", x["present_after_batch"])
    print("   our after batch", y["present_after_batch"])
    for a, b in zip(x["decode"], y["decode"]):
        if a: print("   ref dec keys", [k[:8] for k in a["keys"]], "present", a["present"])
        if b: print("   our dec keys", [k[:8] for k in b["keys"]], "present", b["present"])
