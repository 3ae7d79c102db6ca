"""Host link probe: pinned H2D alone, D2H alone, and both directions at once
(separate streams), plus a chunked D2H of a strided 2-D block the way the
pipelined host path copies output blocks.  GPU box only.
    python tools/pcie_probe.py [GB]
"""
import json
import sys

import torch


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    gb = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
    n = int(gb * (1 << 30)) // 4
    h_in = torch.empty(n, dtype=torch.float32).pin_memory()
    h_out = torch.empty(n, dtype=torch.float32).pin_memory()
    d_a = torch.empty(n, dtype=torch.float32, device="cuda")
    d_b = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    byts = n * 4

    def h2d():
        d_a.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_b, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    # strided 2-D D2H: a [rows, cols] block out of a [rows, ld] matrix
    ld = 20000
    rows = n // ld
    cols = 2560
    d_m = d_b[: rows * ld].view(rows, ld)
    h_m = h_out[: rows * ld].view(rows, ld)

    def d2h_2d():
        for c0 in range(0, ld - cols + 1, cols):
            h_m[:, c0:c0 + cols].copy_(d_m[:, c0:c0 + cols], non_blocking=True)

    # the same blocks through cudaMemcpy2DAsync (what the pipelined host path uses)
    import ctypes
    import glob
    import os

    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                  "libcudart.so*"))
    rt = ctypes.CDLL(libs[0])
    stream = torch.cuda.current_stream().cuda_stream

    def d2h_2d_rt(width_cols=cols):
        for c0 in range(0, ld - width_cols + 1, width_cols):
            e = rt.cudaMemcpy2DAsync(ctypes.c_void_p(h_m.data_ptr() + c0 * 4), ctypes.c_size_t(ld * 4),
                                     ctypes.c_void_p(d_m.data_ptr() + c0 * 4), ctypes.c_size_t(ld * 4),
                                     ctypes.c_size_t(width_cols * 4), ctypes.c_size_t(rows), 2,
                                     ctypes.c_void_p(stream))
            assert e == 0, e

    r = {"bytes": byts}
    r["h2d_GBps"] = byts / timed(h2d) / 1e6
    r["d2h_GBps"] = byts / timed(d2h) / 1e6
    r["both_GBps_total"] = 2 * byts / timed(both) / 1e6
    r["d2h_2d_torch_GBps"] = (rows * (ld // cols) * cols * 4) / timed(d2h_2d) / 1e6
    for w in (256, 1024, 2560, 5120):
        r[f"d2h_2d_memcpy2d_w{w}_GBps"] = (rows * (ld // w) * w * 4) / timed(lambda: d2h_2d_rt(w)) / 1e6
    print(json.dumps(r))


if __name__ == "__main__":
    main()
