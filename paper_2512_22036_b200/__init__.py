"""B200-native Fusco MoE token shuffle (arxiv 2512.22036).

The expert-parallel dispatch/combine path of the reference package
``shuffleforge`` rebuilt for NVLink-5/NVSwitch B200 boxes: an on-device
layout planner, a push dispatch that writes token rows straight into every
owner's expert-major rows (one crossing per token and rank), and a pull
combine fused with the k-ascending weighted reduction — hand-written sm_100a
CUDA behind the C ABI in ``include/fusco.h`` (``lib/libfusco.so``).

Public API (reference names kept, see ``api``):
  run_exchange, build_plan_pair, build_plan, dispatch_loads, dedup_ratio,
  build_dispatch_plan / build_combine_plan / build_direct_plans,
  allocate_buffers, fill_token_buffers, apply_node_level, apply_expert_level,
  run_experts, reduce_outputs, execute_dispatch / execute_combine,
  RoutingAssignment, gen_realworld / gen_single_node / gen_imbalanced,
  ClusterTopology, ExpertPlacement, round_robin_placement, greedy_groups ...
Per-rank multi-GPU API: ``EPBuffer`` (build_plan / dispatch / combine).
"""

from .balancer import greedy_groups, group_load, optimal_groups, static_groups
from .routing import (
    RoutingAssignment,
    derive_token_node,
    gen_imbalanced,
    gen_realworld,
    gen_single_node,
    load_trace,
    local_routing,
    save_trace,
)
from .topology import (
    ClusterTopology,
    ExpertPlacement,
    box,
    load_topology,
    preset,
    round_robin_placement,
    save_topology,
)

__version__ = "0.1.0"

_LAZY = {
    # GPU-side names (import torch + libfusco on first use)
    "run_exchange": "api",
    "execute_exchange": "api",
    "run_baseline": "api",
    "build_plan_pair": "api",
    "build_plan": "api",
    "build_dispatch_plan": "api",
    "build_combine_plan": "api",
    "build_direct_plans": "api",
    "allocate_buffers": "api",
    "fill_token_buffers": "api",
    "apply_node_level": "api",
    "apply_expert_level": "api",
    "run_experts": "api",
    "reduce_outputs": "api",
    "execute_dispatch": "api",
    "execute_combine": "api",
    "dispatch_loads": "api",
    "dedup_ratio": "api",
    "naive_inter_node_bytes": "api",
    "make_token_payloads": "api",
    "identity_expert": "api",
    "scaled_expert": "api",
    "ExchangeResult": "api",
    "PhaseReport": "api",
    "GpuPlan": "api",
    "ActivationLayout": "api",
    "EPBuffer": "engine",
    "EmulatedCluster": "engine",
    "Rank": "engine",
    "Plan": "engine",
    "plan_to_json": "wire",
    "descriptor_to_bytes": "wire",
    "descriptor_from_bytes": "wire",
    "run_matrix": "matrix",
    "BenchConfig": "matrix",
}


def __getattr__(name):
    if name in _LAZY:
        import importlib

        mod = importlib.import_module(f".{_LAZY[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)


__all__ = [
    "ClusterTopology",
    "ExpertPlacement",
    "RoutingAssignment",
    "box",
    "derive_token_node",
    "gen_imbalanced",
    "gen_realworld",
    "gen_single_node",
    "greedy_groups",
    "group_load",
    "load_topology",
    "load_trace",
    "local_routing",
    "optimal_groups",
    "preset",
    "round_robin_placement",
    "save_topology",
    "save_trace",
    "static_groups",
    *sorted(_LAZY),
    "__version__",
]
