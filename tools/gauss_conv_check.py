"""Bit-identity check of the Gauss Gram operand feeds (GPU box only):
PS_GAUSS_CONV=1 (S / D formed in shared memory) against PS_GAUSS_CONV=0
(S / D planes precomputed by gauss_planes_kernel and streamed by TMA).  Both
feeds hand the tensor cores the same fp16 operands, so PLV / iPLV / ciPLV
must agree bit for bit.  Also run with PS_CTA_GROUP=1 for the one-CTA kernel.
    python tools/gauss_conv_check.py
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [  # (N, T, R, seed): ragged N and T (K tail, partial tiles), trials
    (700, 8192, 1, 1),
    (300, 8200, 2, 2),
    (1030, 16384, 1, 3),
]


def child(out_dir):
    import torch

    from paper_1710_08037_b200 import connectivity as C

    for n, t, r, seed in CASES:
        g = np.random.default_rng(seed)
        ph = g.uniform(-np.pi, np.pi, size=(n, t, r))
        amp = g.uniform(0.5, 1.5, size=(n, t, r))
        x = (amp * np.exp(1j * ph)).astype(np.complex64)
        x[: n // 10] = x[n // 10: 2 * (n // 10)] * np.exp(1j * 0.3)  # coupled rows
        xd = torch.from_numpy(np.ascontiguousarray(np.transpose(x, (2, 0, 1)))).cuda().permute(1, 2, 0)
        res = C.plv_family(xd, input_kind="analytic")
        torch.cuda.synchronize()
        for m in ("plv", "iplv", "ciplv"):
            np.save(os.path.join(out_dir, f"{n}_{t}_{r}_{m}.npy"), np.asarray(res[m].values.cpu()))
        print("variant", res["plv"].meta.get("gram_variant"), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2])
        sys.exit(0)
    bad = 0
    for cg in ("2", "1"):
        dirs = {}
        for conv in ("0", "1"):
            d = tempfile.mkdtemp()
            env = dict(os.environ, PS_GAUSS="1", PS_GAUSS_CONV=conv, PS_CTA_GROUP=cg)
            subprocess.run([sys.executable, __file__, "--child", d], env=env, check=True)
            dirs[conv] = d
        for n, t, r, _ in CASES:
            for m in ("plv", "iplv", "ciplv"):
                a = np.load(os.path.join(dirs["0"], f"{n}_{t}_{r}_{m}.npy"))
                b = np.load(os.path.join(dirs["1"], f"{n}_{t}_{r}_{m}.npy"))
                same = np.array_equal(a, b, equal_nan=True)
                diff = float(np.nanmax(np.abs(a - b))) if a.shape == b.shape else float("inf")
                print(f"cta_group={cg} N={n} T={t} R={r} {m}: bit-identical={same} max|diff|={diff:.3e}")
                bad += not same
        # one-trial cases against an fp64 restatement (unit phasors, |Z Z^H| / T)
        for n, t, r, seed in CASES:
            if r != 1:
                continue
            g = np.random.default_rng(seed)
            ph = g.uniform(-np.pi, np.pi, size=(n, t, r))
            g.uniform(0.5, 1.5, size=(n, t, r))
            z = np.exp(1j * ph[:, :, 0])
            z[: n // 10] = z[n // 10: 2 * (n // 10)] * np.exp(1j * 0.3)
            c = (z @ z.conj().T) / t
            for m, ref in (("plv", np.abs(c)), ("iplv", np.abs(c.imag))):
                a = np.load(os.path.join(dirs["1"], f"{n}_{t}_{r}_{m}.npy"))
                err = float(np.max(np.abs(a - ref)))
                print(f"cta_group={cg} N={n} T={t} {m} vs fp64: max|err|={err:.3e}")
                bad += not err <= 1e-5  # the split suite tolerance (tests/test_gpu_parity.py TOL)
    print("gauss_conv_check", "OK" if bad == 0 else f"FAIL ({bad})")
    sys.exit(1 if bad else 0)
