"""GPU micro-benchmark of the b >= 2 one-pass pass kernels (msvd_aw_gram):
the split-role kernel (plain pass and check refresh), with the results
compared bit for bit across repeats and against torch fp64.
    python scripts/bench_split.py [b n m]"""
import os
import subprocess
import sys

CASES = [(4, 500, 500_000), (2, 1000, 1_000_000), (3, 500, 500_000)]
ENVS = [{}, {"MSVD_SPLIT_GROUPS": "4", "MSVD_SPLIT_STAGE_KB": "16"}]


def child(b, n, m):
    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2602_16797_b200 import minsvd

    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(n + b)
    ldp = n + (n & 1)
    a = torch.randn(m, ldp, dtype=torch.float64, device=dev, generator=g)[:, :n]
    w = torch.randn(n, b, dtype=torch.float64, device=dev, generator=g)
    op = minsvd.DeviceDenseOperator(a)
    op.ctx.kernel_paths(reset=True)
    aw0, z0 = op.aw_gram(w)
    paths = sorted(op.ctx.kernel_paths())
    aw_ref = a @ w
    z_ref = a.t() @ aw_ref
    e1 = (aw0 - aw_ref).abs().max().item() / aw_ref.abs().max().item()
    e2 = (z0 - z_ref).abs().max().item() / z_ref.abs().max().item()
    same = True
    for _ in range(3):
        aw, z = op.aw_gram(w)
        same = same and torch.equal(aw, aw0) and torch.equal(z, z0)
    op.ctx.profile(1)
    for _ in range(10):
        op.aw_gram(w)
    ms, cnt = op.ctx.profile_read()["apply"]
    per = ms / cnt
    print(f"b={b} n={n} m={m} paths={paths} {per:.4f} ms/launch = {8e-6 * m * n / per:.0f} GB/s  "
          f"err aw {e1:.1e} z {e2:.1e} repeatable={same}", flush=True)
    # the check-refresh pass (EX): also A^T E
    e = torch.randn(m, b, dtype=torch.float64, device=dev, generator=g)
    op.ctx.profile(0)
    op.ctx.kernel_paths(reset=True)
    awx, zx, zex = op.aw_gram_ex(w, e)
    paths = sorted(op.ctx.kernel_paths())
    ze_ref = a.t() @ e
    e3 = (zex - ze_ref).abs().max().item() / ze_ref.abs().max().item()
    e4 = (zx - z_ref).abs().max().item() / z_ref.abs().max().item()
    op.ctx.profile(1)
    for _ in range(10):
        op.aw_gram_ex(w, e)
    ms, cnt = op.ctx.profile_read()["apply"]
    per = ms / cnt
    print(f"   EX  paths={paths} {per:.4f} ms/launch = {8e-6 * m * n / per:.0f} GB/s  err z {e4:.1e} ze {e3:.1e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
        sys.exit(0)
    cases = CASES
    if len(sys.argv) >= 4:
        cases = [(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]))]
    for b, n, m in cases:
        for env in ENVS:
            e = dict(os.environ)
            e.update(env)
            print(f"--- {env}", flush=True)
            try:
                r = subprocess.run([sys.executable, __file__, "child", str(b), str(n), str(m)], env=e, timeout=120)
                if r.returncode != 0:
                    print(f"    rc={r.returncode}", flush=True)
            except subprocess.TimeoutExpired:
                print("    TIMEOUT (hang)", flush=True)
