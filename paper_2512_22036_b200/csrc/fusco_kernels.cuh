// fusco_kernels.cuh — the three hot-path kernels of the shuffle.
//
//   layout_kernel    on-device planner: per-(rank, expert) counts, offsets,
//                    row_of[t,k], first_mask, dedup statistics
//                    (reference planner.py:126-196, routing.py:86-98)
//   dispatch_kernel  push: token rows -> owners' expert-major rows over NVLink,
//                    one crossing per (token, rank), receiver-side fan-out
//                    (reference engine.py:266-276 dispatch, 799-851)
//   combine_kernel   pull + k-ascending weighted reduction back to token order
//                    (reference engine.py:266-276 combine, 313-338, 967-1049)
//
// All three are persistent cooperative launches; their cross-rank waits are
// split into an explicit REMOTE phase so that P ranks can be emulated on one
// GPU by launching LOCAL for every rank, then REMOTE for every rank.
#pragma once
// Umbrella: layout.cuh (planner), dispatch.cuh (push + fan-out),
// combine.cuh (pull + reduction), probe.cuh (bandwidth probes).
#include "layout.cuh"
#include "dispatch.cuh"
#include "combine.cuh"
#include "probe.cuh"
