"""Device-resident timing sweep of the hot path for one config under several
environment settings (PS_KC_BLOCKS, PS_RASTER, ...).  GPU box only.
    python tools/sweep.py c5 PS_KC_BLOCKS=2,4 PS_RASTER=1,12
"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(cfg, steps=3):
    import numpy as np
    import torch

    from paper_1710_08037_b200 import connectivity as C
    from paper_1710_08037_b200 import workloads as W

    N, T, R, B, dt, kind = W.CONFIGS[cfg]
    x = W.generate(cfg)
    bands = x.ndim == 4
    store = np.ascontiguousarray(np.transpose(x, (2, 0, 1)) if not bands else np.transpose(x, (0, 3, 1, 2)))
    xd = torch.from_numpy(store).cuda()
    xv = xd.permute(1, 2, 0) if not bands else xd.permute(0, 2, 3, 1)
    outs = {m: torch.empty((B, N, N), device="cuda") for m in ("plv", "iplv", "ciplv")}
    for _ in range(2):
        C.plv_family(xv, input_kind=kind, bands=bands, out=outs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = []
    e0.record()
    for _ in range(steps):
        r = C.plv_family(xv, input_kind=kind, bands=bands, out=outs, timing=True)
        st.append((r["plv"].meta["ms_normalize"], r["plv"].meta["ms_gram"], r["plv"].meta["ms_finish"]))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    work = W.pair_samples(N, T, R, B)
    print(json.dumps({"cfg": cfg, "env": {k: os.environ.get(k) for k in os.environ if k.startswith("PS_")},
                      "ms_step": ms, "pair_samples_per_s": work / ms * 1e3,
                      "normalize_ms": float(np.median([s[0] for s in st])),
                      "gram_ms": float(np.median([s[1] for s in st])),
                      "finish_ms": float(np.median([s[2] for s in st])),
                      "refined": int(r["plv"].meta["n_refined_pairs"])}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], steps=int(os.environ.get("SWEEP_STEPS", "3")))
        sys.exit(0)
    cfg = sys.argv[1]
    axes = []
    for a in sys.argv[2:]:
        k, vs = a.split("=", 1)
        sep = ";" if ";" in vs else ","  # values with commas (PS_LOCKSTEP=32,2;16,1)
        axes.append([(k, v) for v in vs.split(sep)])
    for combo in itertools.product(*axes) if axes else [()]:
        env = dict(os.environ)
        env.update(dict(combo))
        subprocess.run([sys.executable, __file__, "--child", cfg], env=env, check=False)
