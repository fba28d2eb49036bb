"""Multi-GPU DGSM build and query.

The path shards naturally:
  * lights are independent (one atlas per light)           -> light groups;
  * tau is a sum over Gaussians (Eq.2) -> within a group,
    Gaussians are split into contiguous shards, every rank builds the partial
    optical depth of its shard (DGSM_OUTPUT_TAU), the partials are summed by a
    reduce-scatter over the shell axis K (NCCL over NVLink; NVLS where NCCL
    picks it), and each rank applies Eq.4 (T = exp(-tau)) to the K/g shells it
    owns (dgsm_exp_epilogue).
  * query: the product over lights (Q13) is an all-reduce(PRODUCT) of the
    per-light receiver transmittances.

Binning is per Gaussian (its tiles depend on it alone), so a shard's binned
lists are exactly the full lists restricted to the shard: the reduce-scattered
tau equals the unsharded build's tau up to fp32 summation order.

One process per GPU; torch.distributed supplies the process groups and the
collectives.  The build/exp functions are parameters so the host logic can be
exercised on CPU (gloo) in tests; the product path uses the CUDA library.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


@dataclasses.dataclass
class Layout:
    """Assignment of lights and Gaussian shards to ranks.

    groups[j]      ranks of group j (consecutive ranks);
    lights_of[j]   lights built by group j;
    Every light belongs to exactly one group.  Group size g > 1 only when
    there are fewer lights than ranks; then K must be divisible by g."""
    world: int
    groups: List[List[int]]
    lights_of: List[List[int]]

    def group_index(self, rank: int) -> int:
        for j, g in enumerate(self.groups):
            if rank in g:
                return j
        return -1

    def shard_of(self, rank: int) -> Tuple[int, int]:
        """(index within its group, group size)."""
        j = self.group_index(rank)
        if j < 0:
            return 0, 1
        return self.groups[j].index(rank), len(self.groups[j])


def plan_layout(n_lights: int, world: int, light_cost: Optional[Sequence[float]] = None) -> Layout:
    """Lights >= ranks: light-parallel, lights dealt to ranks by longest-processing-
    time first on `light_cost` (e.g. per-light key counts), no communication.
    Lights < ranks: floor(world / L) consecutive ranks per light (Gaussian-sharded);
    leftover ranks join the first groups round-robin."""
    if n_lights < 1 or world < 1:
        raise ValueError("need >= 1 light and >= 1 rank")
    if n_lights >= world:
        cost = list(light_cost) if light_cost is not None else [1.0] * n_lights
        order = sorted(range(n_lights), key=lambda l: (-cost[l], l))
        load = [0.0] * world
        lights_of: List[List[int]] = [[] for _ in range(world)]
        for l in order:
            r = min(range(world), key=lambda q: (load[q], q))
            lights_of[r].append(l)
            load[r] += cost[l]
        for x in lights_of:
            x.sort()
        return Layout(world, [[r] for r in range(world)], lights_of)
    g = world // n_lights
    extra = world - g * n_lights
    groups, r = [], 0
    for l in range(n_lights):
        size = g + (1 if l < extra else 0)
        groups.append(list(range(r, r + size)))
        r += size
    return Layout(world, groups, [[l] for l in range(n_lights)])


def shard_range(n: int, index: int, size: int) -> Tuple[int, int]:
    """Contiguous, balanced range of Gaussians for shard `index` of `size`."""
    base, rem = divmod(n, size)
    start = index * base + min(index, rem)
    return start, start + base + (1 if index < rem else 0)


def make_groups(layout: Layout, backend_group=None) -> List[Optional[dist.ProcessGroup]]:
    """One process group per multi-rank light group (collective: all ranks call it)."""
    out = []
    for g in layout.groups:
        out.append(dist.new_group(ranks=g) if len(g) > 1 else None)
    return out


BuildFn = Callable[..., torch.Tensor]


def build_sharded(gaussians: Dict[str, torch.Tensor], lights: Dict[str, np.ndarray], res: int, K: int,
                  layout: Layout, pgroups: List[Optional[dist.ProcessGroup]], build_fn: BuildFn,
                  exp_fn: Callable[[torch.Tensor], torch.Tensor], gather: bool = True,
                  **build_kw) -> Dict[int, torch.Tensor]:
    """Build the atlases of this rank's lights.

    build_fn(gaussians_shard, lights_subset, res, K, output_tau=bool, **build_kw) -> [L', K, H, W]
    exp_fn(tau) -> exp(-tau)   (dgsm_exp_epilogue on the GPU)

    Returns {light: tensor}: with gather=True the full [K, H, W] transmittance of
    each of this rank's lights (all-gather of the owned shell chunks); with
    gather=False the owned chunk [K/g, H, W] only."""
    rank = dist.get_rank() if dist.is_initialized() else 0
    j = layout.group_index(rank)
    if j < 0:
        return {}
    my_lights = layout.lights_of[j]
    idx, g = layout.shard_of(rank)
    pos = np.asarray(lights["position"], np.float32).reshape(-1, 3)
    tm = np.asarray(lights["t_max"], np.float32).reshape(-1)
    sub = dict(position=pos[my_lights], t_max=tm[my_lights])
    if g == 1:
        T = build_fn(gaussians, sub, res, K, output_tau=False, **build_kw)
        return {l: T[q] for q, l in enumerate(my_lights)}
    if K % g:
        raise ValueError(f"K={K} must be divisible by the group size {g} for the shell reduce-scatter")
    n = next(iter(gaussians.values())).shape[0]
    s0, s1 = shard_range(n, idx, g)
    shard = {k: v[s0:s1] for k, v in gaussians.items()}
    tau = build_fn(shard, sub, res, K, output_tau=True, **build_kw)       # partial optical depth
    out = {}
    kc = K // g
    for q, l in enumerate(my_lights):
        full = tau[q].contiguous()                                      # [K, H, W]
        mine = torch.empty((kc,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
        dist.reduce_scatter_tensor(mine, full, op=dist.ReduceOp.SUM, group=pgroups[j])
        T_mine = exp_fn(mine)                                           # Eq.4 on the owned shells
        if gather:
            T_full = torch.empty_like(full)
            dist.all_gather_into_tensor(T_full, T_mine, group=pgroups[j])
            out[l] = T_full
        else:
            out[l] = T_mine
    return out


def query_combine(T_local: torch.Tensor, group=None) -> torch.Tensor:
    """Product over lights held by different ranks (Q13): all-reduce(PRODUCT)
    of per-rank partial products (ranks without lights contribute 1)."""
    dist.all_reduce(T_local, op=dist.ReduceOp.PRODUCT, group=group)
    return T_local


def query_sharded(atlases: Dict[int, torch.Tensor], lights: Dict[str, np.ndarray], positions: torch.Tensor,
                  layout: Layout, query_fn: Callable[..., torch.Tensor]) -> torch.Tensor:
    """T(x) = prod_l T_l(x): each group's first rank queries its lights' atlases,
    then all ranks all-reduce(PRODUCT).  query_fn(atlas [L',K,H,W], lights_subset, positions) -> [m]."""
    rank = dist.get_rank() if dist.is_initialized() else 0
    j = layout.group_index(rank)
    m = positions.shape[0]
    T = torch.ones(m, dtype=torch.float32, device=positions.device)
    if j >= 0 and layout.groups[j][0] == rank and atlases:
        ls = sorted(atlases)
        pos = np.asarray(lights["position"], np.float32).reshape(-1, 3)
        tm = np.asarray(lights["t_max"], np.float32).reshape(-1)
        sub = dict(position=pos[ls], t_max=tm[ls])
        at = torch.stack([atlases[l] for l in ls]).contiguous()
        T = query_fn(at, sub, positions)
    if dist.is_initialized() and dist.get_world_size() > 1:
        T = query_combine(T)
    return T


# ---------------------------------------------------------------- CUDA path
def cuda_build_fn(gaussians, lights, res, K, output_tau=False, **kw):
    from . import dgsm
    opts = dgsm.Options(output_tau=output_tau, **kw)
    return dgsm.build(gaussians, lights, res, K, opts)


def cuda_exp_fn(tau):
    from . import dgsm
    return dgsm.exp_epilogue(tau.contiguous(), out=tau.contiguous())


def cuda_query_fn(atlas, lights, positions):
    from . import dgsm
    return dgsm.query(atlas, lights, positions)
