"""GPU micro-benchmark of the sketch S A (msvd_sketch) at BASELINE shapes, by the pacing
window of the slice gather (MSVD_SKETCH_WIN_LOG2; 0 = unpaced).  Prints the time per call and a checksum of SA's bytes (all variants must agree).
    python scripts/bench_sketch.py"""
import ctypes as C
import hashlib
import os
import subprocess
import sys

CASES = [(1_000_000, 1000, 4000), (500_000, 500, 2000), (1_000_000, 500, 1000), (10_000, 100, 200)]
ENVS = [{}]


def child(m, n, d):
    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2602_16797_b200 import minsvd

    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(n)
    a = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
    op = minsvd.DeviceDenseOperator(a)
    sa = torch.empty((n, d), dtype=torch.float64, device=dev)
    call = lambda: minsvd.check(minsvd.lib().msvd_sketch(op.handle, d, 4, 99, C.c_void_p(sa.data_ptr())))
    call()
    h = hashlib.sha256(sa.cpu().numpy().tobytes()).hexdigest()[:16]
    op.ctx.profile(True)
    for _ in range(5):
        call()
    ms, cnt = op.ctx.profile_read()["sketch"]
    per = ms / 5
    print(f"m={m} n={n} d={d}: {per:.3f} ms per sketch = {8e-6 * m * n / per:.0f} GB/s algorithmic; sha {h}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
        sys.exit(0)
    for m, n, d in CASES:
        for env in ENVS:
            e = dict(os.environ)
            e.update(env)
            print(f"--- {env}", flush=True)
            try:
                subprocess.run([sys.executable, __file__, "child", str(m), str(n), str(d)], env=e, timeout=180)
            except subprocess.TimeoutExpired:
                print("    TIMEOUT", flush=True)
