# round 2 (session 3), call 10 (2 GPUs): decode timeline with the sender-side block-release stamp
set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522"
for kv in BASE=1 FUSCO_BALANCE=0 FUSCO_DBG_BLK=1; do
  env $kv TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py dsv3_decode warp tma > gpurun_out/e10_trace.log 2>&1; echo "== $kv"; grep -A21 "rank 0\]" gpurun_out/e10_trace.log | grep -E "dispatch|combine|layout.end|last"; grep -A21 "rank 1\]" gpurun_out/e10_trace.log | grep -E "dispatch|combine.ready"
done
for kv in BASE=1 FUSCO_DBG_BLK=1; do
  env $kv TRACE_GRAPH=1 timeout 200 $TR tools/trace_step.py mixtral warp tma > gpurun_out/e10_trace.log 2>&1; echo "== mixtral $kv"; grep -A21 "rank 0\]" gpurun_out/e10_trace.log | grep -E "dispatch|combine"
done
