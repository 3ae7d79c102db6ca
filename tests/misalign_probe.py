import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from oracle import plv_oracle as O
from paper_1710_08037_b200 import connectivity as C
rng = np.random.default_rng(3)
for T in (4096, 1000, 2048, 999):
    for kind, dt in (("real", np.float32), ("real", np.float64), ("analytic", np.complex64), ("analytic", np.complex128)):
        for c0 in (1, 3):
            N = 9
            if np.issubdtype(dt, np.complexfloating):
                buf = (rng.standard_normal((N, T + 8)) + 1j * rng.standard_normal((N, T + 8))).astype(dt)
            else:
                buf = rng.standard_normal((N, T + 8)).astype(dt)
            x = buf[:, c0:c0 + T]
            xd = torch.from_numpy(buf).cuda()[:, c0:c0 + T]
            ref = O.plv_family(x[:, :, None].astype(np.complex128 if kind == "analytic" else np.float64), input_kind=kind)
            for prec, tol in (("split", 1e-5), ("fp64", 1e-12 if dt in (np.float64, np.complex128) else 1e-5)):
                res = C.plv_family(xd[:, :, None], input_kind=kind, precision=prec)
                err = max(float(np.max(np.abs(res[m].values.double().cpu().numpy() - ref[m]))) for m in ("plv", "iplv", "ciplv"))
                status = "ok" if err <= tol else "FAIL"
                print(T, kind, np.dtype(dt).name, c0, prec, f"{err:.2e}", status, flush=True)
