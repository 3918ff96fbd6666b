# round 2 (session 3), call 14 (2 GPUs): P>1 push unit size / grid sweep
set -x
for cfg in mixtral dsv3; do
  for kv in BASE=1 FUSCO_LIB=_ab/libs/u16.so FUSCO_LIB=_ab/libs/u4.so FUSCO_DISP_CTAS=1 FUSCO_DISP_CTAS=2 "FUSCO_LIB=_ab/libs/u4.so FUSCO_DISP_CTAS=2"; do
    env $kv timeout 120 python tools/push_probe.py --config $cfg --gpus 2 --iters 15 --tag "$kv" 2>&1 | tail -1
  done
done > gpurun_out/e14_probe.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/e14_probe.jsonl'):
    if not l.startswith('{'): print(l.strip()[:200]); continue
    d=json.loads(l); print(d['config'], d['tag'][:40].ljust(40), d['us'], 'push', d['push_gbps'])
PY
timeout 120 python tools/p2p_probe.py 64 > gpurun_out/e14_p2p1.json 2>&1; tail -1 gpurun_out/e14_p2p1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29670 tools/p2p_probe.py 64 > gpurun_out/e14_p2p.json 2>&1; tail -1 gpurun_out/e14_p2p.json
