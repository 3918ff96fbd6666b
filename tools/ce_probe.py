"""Copy-engine peer-copy rates (single process, 2 GPUs, both directions at once):
one large copy vs many 1-2 MB segments, to judge a CE-based pull."""
import torch

assert torch.cuda.device_count() >= 2
n = 256 << 20
src = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}") for d in range(2)]
dst = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}") for d in range(2)]
streams = [torch.cuda.Stream(device=f"cuda:{d}") for d in range(2)]


def bench(seg, reps=5):
    def go():
        for d in range(2):  # device d pulls from the other device
            with torch.cuda.stream(streams[d]):
                o = 1 - d
                for off in range(0, n, seg):
                    dst[d][off:off + seg].copy_(src[o][off:off + seg], non_blocking=True)
    go()
    for d in range(2):
        torch.cuda.synchronize(d)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2)]
    for d in range(2):
        ev[d][0].record(streams[d])
    for _ in range(reps):
        go()
    for d in range(2):
        ev[d][1].record(streams[d])
    for d in range(2):
        torch.cuda.synchronize(d)
    ms = max(ev[d][0].elapsed_time(ev[d][1]) for d in range(2)) / reps
    return n / (ms * 1e-3) / 1e9


for seg in (n, 16 << 20, 2 << 20, 1 << 20, 256 << 10):
    print(f"segment {seg >> 10:7d} KiB: {bench(seg):7.1f} GB/s per direction (both directions busy)")
