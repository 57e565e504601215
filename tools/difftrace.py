import sys, json
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import scenarios as S, oracle
from paper_2510_09665_b200.api import Engine
C = oracle.C()
for fn in (S.sc_random_trace_roomy, S.sc_random_trace_evicting, S.sc_random_trace_pinned,
           S.sc_random_trace_blocking, S.sc_random_trace_decode):
    ref = json.loads(json.dumps(fn(oracle.RefEngine, C)))
    got = json.loads(json.dumps(fn(Engine, C)))
    print(fn.__name__, "equal:", ref == got)
    for t, (a, b) in enumerate(zip(ref, got)):
        for i, (x, y) in enumerate(zip(a, b)):
            if x != y:
                for k in x:
                    if x[k] != y[k]:
                        if k == "results":
                            print(" trace", t, "iter", i, "codes ref:", [[c for _, c in q] for q in x[k]],
                                  "ours:", [[c for _, c in q] for q in y[k]])
                        else:
                            print(" trace", t, "iter", i, k, "ref:", str(x[k])[:200], "ours:", str(y[k])[:200])
                break
