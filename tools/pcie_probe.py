"""PCIe copy rates with pinned host buffers: H2D alone, D2H alone, both concurrently."""
import torch

n = 64 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(f, reps=20):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    for _ in range(reps):
        f()
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


for name, f in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timeit(f)
    print(f"{name}: {ms:.3f} ms per 64 MiB -> {n / ms / 1e6:.1f} GB/s per direction")
for chunks in (4, 16):
    c = n // chunks

    def h2d_c():
        with torch.cuda.stream(s1):
            for i in range(chunks):
                d1[i * c:(i + 1) * c].copy_(h1[i * c:(i + 1) * c], non_blocking=True)
    ms = timeit(h2d_c)
    print(f"h2d {chunks} chunks: {n / ms / 1e6:.1f} GB/s")
