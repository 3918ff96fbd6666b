"""Per-rank worker for the real multi-GPU parity test (launched by torchrun
from tests/test_gpu_multiproc.py).  Every rank runs the production path
(EPBuffer: CUDA-IPC symmetric regions, FS_PHASE_ALL kernels synchronising
over NVLink flags) and checks its own slice against the oracle."""

import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import shuffle_oracle as O  # noqa: E402
from paper_2512_22036_b200 import EPBuffer, box, gen_realworld, round_robin_placement  # noqa: E402
from paper_2512_22036_b200.baseline import DisaggregatedShuffle  # noqa: E402


def main() -> int:
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P, rank = dist.get_world_size(), dist.get_rank()
    E, K = int(os.environ.get("MP_E", 64)), int(os.environ.get("MP_K", 8))
    T_l = int(os.environ.get("MP_T", 256))  # tokens per rank (BASELINE sizes: 4096 / 8192)
    iters = int(os.environ.get("MP_ITERS", 4))
    big = T_l > 1024  # full-size check: activations on the device, combine on sampled tokens
    H = int(os.environ.get("MP_H", 2048))
    dt = os.environ.get("MP_DT", "bf16")
    topo = box(P)
    pl = round_robin_placement(E, topo)
    buf = EPBuffer(num_experts=E, topk=K, hidden=H, dtype=dt, max_tokens=T_l, timeout_ms=20000)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    base = DisaggregatedShuffle(num_experts=E, topk=K)
    dev = torch.device("cuda", local)
    failures = 0
    for it in range(iters):
        a = gen_realworld(P * T_l, K, topo, pl, seed=10 + it, zipf_s=0.4 * it)
        vals = np.random.default_rng(it).standard_normal((a.num_tokens, H)).astype(np.float32)
        payload = O.encode(vals, dt)
        ids = np.flatnonzero(a.source == rank)
        x = torch.as_tensor(payload[ids], device=dev).view(tdt).contiguous()
        idx = torch.as_tensor(a.experts[ids], device=dev)
        w = torch.as_tensor(a.weights[ids], dtype=torch.float64, device=dev)
        plan = buf.build_plan(idx)
        act = buf.dispatch(x, plan)
        rows = plan.num_rows
        if it % 2:  # exercise the act_out contract: expert writes into the symmetric buffer
            buf.expert_out(rows).copy_(act[:rows])
            out = buf.combine(plan, w, src="act_out", acc="f64")
        else:
            out = buf.combine(plan, w, src="act", acc="f64")
        buf.check()
        # the same shuffle with the router weights at dispatch and fp32
        # accumulation: the owners pre-reduce groups of a token's rows
        # (production P > 1 path), within the stated tolerance
        w32 = w.float().contiguous()
        plan32 = buf.build_plan(idx)
        act32 = buf.dispatch(x, plan32, topk_w=w32)
        out32 = buf.combine(plan32, w32, src="act", acc="f32")
        buf.check()
        tol = dict(rtol=2.0**-8, atol=1e-3) if dt == "bf16" else dict(rtol=1e-5, atol=1e-6)
        layouts, row_of = O.activation_layouts(a.experts, a.source, pl.owner, P)
        if not np.array_equal(plan.row_of.cpu().numpy(), row_of[ids]):
            print(f"[rank {rank}] iter {it}: row_of mismatch", flush=True)
            failures += 1
        if big:
            # oracle dispatch evaluated on the device: row r holds token_ids[r]'s payload
            pay_d = torch.as_tensor(payload, device=dev)
            want_act = O.dispatch(pay_d, {rank: layouts[rank]})[rank]
            if not torch.equal(act[:rows].contiguous().view(torch.uint8).reshape(rows, -1), want_act):
                print(f"[rank {rank}] iter {it}: activation mismatch", flush=True)
                failures += 1
            # identity expert: every staged row of token t is x_t; oracle reduction on 1024 sampled tokens
            loc = np.sort(np.random.default_rng(it).choice(ids.size, size=min(ids.size, 1024), replace=False))
            t = ids[loc]
            want = O.reduce_rows(lambda k: payload[t], a.weights[t], dt)
            got = out.view(torch.uint8).reshape(ids.size, -1)[torch.as_tensor(loc, device=dev)].cpu().numpy()
            if not np.array_equal(got, want):
                print(f"[rank {rank}] iter {it}: output mismatch", flush=True)
                failures += 1
            got32 = out32.view(torch.uint8).reshape(ids.size, -1)[torch.as_tensor(loc, device=dev)].cpu().numpy()
            if not np.allclose(O.decode(got32, dt), O.decode(want, dt), **tol):
                print(f"[rank {rank}] iter {it}: fp32 (owner pre-reduced) output out of tolerance", flush=True)
                failures += 1
            del pay_d
            continue
        acts = O.dispatch(payload, layouts)
        got_act = act[:rows].contiguous().view(torch.uint8).cpu().numpy().reshape(rows, -1)
        if not np.array_equal(got_act, acts[rank]):
            print(f"[rank {rank}] iter {it}: activation mismatch", flush=True)
            failures += 1
        want = O.combine(acts, row_of, a.experts, a.weights, pl.owner, ids, dt)
        if not np.array_equal(out.view(torch.uint8).cpu().numpy(), want):
            print(f"[rank {rank}] iter {it}: output mismatch", flush=True)
            failures += 1
        if not np.allclose(O.decode(out32.view(torch.uint8).cpu().numpy(), dt), O.decode(want, dt), **tol):
            print(f"[rank {rank}] iter {it}: fp32 (owner pre-reduced) output out of tolerance", flush=True)
            failures += 1
        # disaggregated NCCL baseline: same activation bytes, outputs within bf16 tolerance
        bact, st = base.dispatch(x, idx)
        if not torch.equal(bact.view(torch.uint8), act[:rows].view(torch.uint8)):
            print(f"[rank {rank}] iter {it}: baseline activation differs from fused", flush=True)
            failures += 1
        bout = base.combine(bact, st, w.float())
        ref = torch.as_tensor(O.decode(want, dt), device=dev)
        if not torch.allclose(bout.float(), ref, **tol):
            print(f"[rank {rank}] iter {it}: baseline output out of tolerance", flush=True)
            failures += 1
    t = torch.tensor([failures], device=dev)
    dist.all_reduce(t)
    buf.close()
    dist.destroy_process_group()
    if rank == 0:
        print(f"multi-GPU parity: world={P} failures={int(t.item())}", flush=True)
    return 0 if int(t.item()) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
