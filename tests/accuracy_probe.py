"""Accuracy probe of the split path vs the fp64 oracle for several TMEM
chunk lengths (PS_KC_BLOCKS); run on the GPU box.  Prints one line per case."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(case):
    import numpy as np

    from oracle import plv_oracle as O
    from paper_1710_08037_b200 import connectivity as C
    from paper_1710_08037_b200 import workloads as W

    if case == "c1":
        x, kind = W.c1(), "real"
    elif case == "c3s":
        x, kind = W.c3(n_signals=256, n_samples=65536), "real"
    elif case == "c5s":
        x, kind = W.c5(n_signals=512, n_samples=16384, n_latent=8), "analytic"
    elif case == "c2s":
        x, kind = W.c2(n_signals=300, n_samples=10000, n_trials=4, n_coupled=30), "real"
    ref = O.plv_family(x, input_kind=kind)
    res = C.plv_family(x, input_kind=kind, precision="split")
    out = {"case": case, "kc_blocks": os.environ.get("PS_KC_BLOCKS", "4"), "gauss": os.environ.get("PS_GAUSS"),
           "gram_variant": int(res["plv"].meta["gram_variant"])}
    for m in ("plv", "iplv", "ciplv"):
        d = np.asarray(res[m].values, dtype=np.float64) - ref[m]
        out[m] = float(np.max(np.abs(d)))
        out[m + "_mean"] = float(np.mean(d))
    out["illcond"] = int(res["plv"].meta["n_refined_pairs"])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2:
        one(sys.argv[2])
        sys.exit(0)
    # `accuracy_probe.py gauss`: the Gauss 3-product Gram (PS_GAUSS=1) around
    # its default chunk (kc 16 = 512 samples); otherwise the 4-product Gram
    gauss = len(sys.argv) > 1 and sys.argv[1] == "gauss"
    kcs = ("4", "8", "16", "32") if gauss else ("1", "2", "4", "8", "100000")
    for case in ("c1", "c5s", "c3s", "c2s"):
        for kc in kcs:
            # PS_KC_UNSAFE: the library caps PS_KC_BLOCKS at the validated chunk otherwise
            env = dict(os.environ, PS_KC_BLOCKS=kc, PS_KC_UNSAFE="1", PS_GAUSS="1" if gauss else "0")
            subprocess.run([sys.executable, __file__, "one", case], env=env, check=False)
