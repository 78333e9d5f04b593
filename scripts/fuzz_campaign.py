"""One-off fuzz campaign: many seeds of tests/test_fuzz_gpu.py's draws (normal
and large), alone and grouped, random forced orientation; prints failures
(problem names) and keeps going. SEEDS=a:b, LARGE=1 for the large draw."""
import os, random, sys, traceback
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
from test_fuzz_gpu import _draw, _draw_large, _check
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner
a, b = (int(x) for x in os.environ.get("SEEDS", "200:240").split(":"))
draw = _draw_large if os.environ.get("LARGE") else _draw
n = 8 if os.environ.get("LARGE") else 24
fails = 0
planner = Planner()
for seed in range(a, b):
    rng = random.Random(seed)
    g = torch.Generator(device="cpu").manual_seed(seed)
    probs = [draw(rng, g, "cuda") for _ in range(n)]
    orient = rng.choice([-1, -1, 0, 1])
    recs = planner.plan([p["inst"] for p in probs])
    for mode in ("alone", "grouped"):
        try:
            if mode == "alone":
                for p, r in zip(probs, recs):
                    ex = Executable([gemm_desc(p["A"], p["B"], p["C"], p["b_layout"], orientation=orient, bias=p["bias"],
                                               activation=p["act"])], [r.program], p["keep"])
                    ex.launch(); torch.cuda.synchronize(); _check(p, f"seed {seed} alone o={orient}"); ex.close()
            else:
                for p in probs: p["C_base"].fill_(float("nan"))
                ex = Executable([gemm_desc(p["A"], p["B"], p["C"], p["b_layout"], orientation=orient, bias=p["bias"],
                                           activation=p["act"]) for p in probs], [r.program for r in recs],
                                [t for p in probs for t in p["keep"]])
                ex.launch(); torch.cuda.synchronize()
                for p in probs: _check(p, f"seed {seed} grouped o={orient}")
                ex.close()
        except AssertionError as e:
            fails += 1
            print("FAIL", e, flush=True)
        except Exception as e:
            fails += 1
            print("ERROR seed", seed, mode, type(e).__name__, str(e)[:200], flush=True)
            sys.exit(1)  # a device fault poisons the context
print(f"seeds {a}..{b}: {fails} failures", flush=True)
