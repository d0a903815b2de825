"""Dev tool: per-chunk timeline of the host pipeline (H2D -> kernel -> D2H on
three streams), rebuilt in Python with torch streams and events around every
copy and kernel, to see where the e2e step loses time against the PCIe
floor.  Prints, per chunk count, the step time and each op's start/end (us)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt

n = 1 << 24
x = (torch.randn(n) * 2).to(torch.bfloat16).pin_memory()
y = torch.empty_like(x).pin_memory()
dx = torch.empty_like(x, device="cuda")
dy = torch.empty_like(x, device="cuda")
S = [torch.cuda.Stream() for _ in range(3)]
main = torch.cuda.current_stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


def step(sizes, evs=None):
    f = ev(); f.record(main)
    for s in S:
        s.wait_event(f)
    off = 0
    for k, c in enumerate(sizes):
        sl = slice(off, off + c)
        e = [ev() for _ in range(6)] if evs is not None else None
        with torch.cuda.stream(S[0]):
            if e: e[0].record()
            dx[sl].copy_(x[sl], non_blocking=True)
            i = ev(); i.record()
            if e: e[1].record()
        S[1].wait_event(i)
        with torch.cuda.stream(S[1]):
            if e: e[2].record()
            kt.ktanh_bf16(dx[sl], out=dy[sl])
            cdone = ev(); cdone.record()
            if e: e[3].record()
        S[2].wait_event(cdone)
        with torch.cuda.stream(S[2]):
            if e: e[4].record()
            y[sl].copy_(dy[sl], non_blocking=True)
            if e: e[5].record()
        if e: evs.append(e)
        off += c
    for s in S:
        j = ev(); j.record(s); main.wait_event(j)


def plan(nch, ramp=False):
    if not ramp:
        c = n // nch
        return [c] * nch
    c = n // nch
    out, cur, left = [], c // 8, n
    while left > 0:
        t = min(cur, left)
        out.append(t); left -= t; cur = min(c, cur * 2)
    return out


for nch in (4, 8, 16, 32, 64):
    for ramp in (False, True):
        sizes = plan(nch, ramp)
        for _ in range(3): step(sizes)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(main)
        for _ in range(10): step(sizes)
        b.record(main); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"chunks={nch:3d} ramp={int(ramp)} n_ops={len(sizes):3d}: {ms:.4f} ms/step {n / ms / 1e6:.2f} Gelem/s", flush=True)

sizes = plan(8)
evs = []
t0 = ev(); t0.record(main)
step(sizes, evs)
torch.cuda.synchronize()
print("timeline, 8 chunks (us from step start): H2D [s,e]  K [s,e]  D2H [s,e]")
for k, e in enumerate(evs):
    r = [t0.elapsed_time(q) * 1e3 for q in e]
    print(f"  {k:2d}: H2D {r[0]:7.1f} {r[1]:7.1f}  K {r[2]:7.1f} {r[3]:7.1f}  D2H {r[4]:7.1f} {r[5]:7.1f}")
