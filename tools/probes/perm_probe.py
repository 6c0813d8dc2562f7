"""Probe: what a random original-order gather / scatter of N doubles costs on
this GPU, cold vs with the source (gather) or destination (scatter) brought
into L2 first -- the K0 / K4 question.  torch ops only;
the numbers bound what a hand-written K0 / K4 can reach.

    python tools/probes/perm_probe.py [N]
"""
import sys

import torch


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)  # evict L2
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
    g = torch.Generator(device="cuda").manual_seed(1)
    perm = torch.randperm(n, device="cuda", generator=g)
    q = torch.randn(n, dtype=torch.float64, device="cuda")
    out = torch.empty_like(q)
    gb = n * 8 / 1e9
    t_copy = timed(lambda: out.copy_(q))
    t_g = timed(lambda: torch.index_select(q, 0, perm, out=out))
    t_gw = timed(lambda: (q.sum(), torch.index_select(q, 0, perm, out=out)))
    t_sum = timed(lambda: q.sum())
    t_s = timed(lambda: out.index_copy_(0, perm, q))
    t_sw = timed(lambda: (out.zero_(), out.index_copy_(0, perm, q)))
    t_zero = timed(lambda: out.zero_())
    print(f"N={n}: copy {t_copy * 1e3:.1f} us ({2 * gb / t_copy * 1e3:.0f} GB/s)")
    print(f"gather cold {t_g * 1e3:.1f} us; with q.sum() first {t_gw * 1e3:.1f} us "
          f"(sum alone {t_sum * 1e3:.1f} us)")
    print(f"scatter cold {t_s * 1e3:.1f} us; with out.zero_() first {t_sw * 1e3:.1f} us "
          f"(zero alone {t_zero * 1e3:.1f} us)")


if __name__ == "__main__":
    main()
