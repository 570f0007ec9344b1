"""PCIe ceiling of the e2e leg: pinned H2D alone, D2H alone, both at once on
two streams (the copy engines are full duplex if the last is ~max of the two),
at the cfg5 per-call volumes (7.43 GB up, 5.40 GB down) and as many chunks."""
import sys
import torch

up, down = 7429160960, 5400166400
nchunk = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def bufs(total):
    n = total // 4 // nchunk
    h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(nchunk)]
    d = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(nchunk)]
    return h, d


hu, du = bufs(up)
hd, dd = bufs(down)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        for h, d in zip(hu, du):
            d.copy_(h, non_blocking=True)


def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        for h, d in zip(hd, dd):
            h.copy_(d, non_blocking=True)


for rep in range(3):
    t1 = timed(h2d)
    t2 = timed(d2h)
    t3 = timed(lambda: (h2d(), d2h()))
    print(f"rep {rep}: H2D {t1:.1f} ms ({up / t1 / 1e6:.1f} GB/s)  D2H {t2:.1f} ms ({down / t2 / 1e6:.1f} GB/s)  "
          f"both {t3:.1f} ms ({(up + down) / t3 / 1e6:.1f} GB/s)")
