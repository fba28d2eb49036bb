"""Multi-GPU DGSM build and query.

The path shards naturally:
  * lights are independent (one atlas per light)           -> light groups;
  * tau is a sum over Gaussians (Eq.2) -> within a group,
    Gaussians are split into contiguous shards, every rank builds the partial
    optical depth of its shard for the group's lights (DGSM_OUTPUT_TAU), the
    partials are summed by ONE reduce-scatter over the group's flattened
    (light, shell) planes (NCCL over NVLink / NVSwitch; NVLS where NCCL picks
    it), and each rank applies Eq.4 (T = exp(-tau), dgsm_exp_epilogue) to the
    planes it owns;
  * query: a rank samples the shell chunks it holds (dgsm_query_chunks: the
    trilinear sample is linear in the atlas, so taps on shells held elsewhere
    count 0); a light whose shells are spread over several ranks is summed by
    an all-reduce(SUM) of N_q floats inside its group; the product over lights
    (Q13) is an all-reduce(PRODUCT) of N_q floats over all ranks.  No atlas is
    ever all-gathered.

Layouts (plan_layout):
  * "light"    (default when lights >= ranks): lights dealt to ranks by
               longest-processing-time on their cost (per-light key counts P_l
               from a replicated plan): no build communication;
  * "shells"   (default when lights < ranks): floor(world / L) consecutive ranks
               per light, Gaussian-sharded, reduce-scatter over the shell axis
               (K divisible by the group size);
  * "gaussian" (BASELINE cfg5's "Gaussians sharded with optical-depth
               reduce-scatter"): ONE group of all ranks building all lights on
               a 1/world Gaussian shard each; the reduce-scatter over the
               [L][K] planes hands each rank L*K/world planes (one light each
               at L = world).  It balances the build exactly but moves
               (world-1)/world of the whole L*K*H*W atlas over NVLink (14 GiB
               per rank at cfg5): DESIGN.md §9 compares the two.

Binning is per Gaussian (its tiles depend on it alone), so a shard's binned
lists are exactly the full lists restricted to the shard: the reduce-scattered
tau equals the unsharded build's tau up to fp32 summation order.

One process per GPU; torch.distributed supplies the process groups and the
collectives.  The build / exp / query functions are parameters so that the
host logic runs on CPU (gloo) in tests with the oracle; the product path uses
the CUDA library (cuda_* below) through the same functions.
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
    lights_of[j]   lights built by group j (every light in exactly one group).
    Within group j (size g) the flattened planes (q, k) -> q*K + k of its
    lights are split into g equal contiguous chunks, chunk i owned by
    groups[j][i] (g = 1: the rank owns everything)."""
    world: int
    groups: List[List[int]]
    lights_of: List[List[int]]
    K: int
    mode: str = "light"

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

    def planes_of(self, rank: int) -> Tuple[int, int]:
        """[p0, p1): the flattened (light-in-group, shell) planes owned by rank."""
        j = self.group_index(rank)
        if j < 0:
            return 0, 0
        i, g = self.shard_of(rank)
        total = len(self.lights_of[j]) * self.K
        c = total // g
        return i * c, (i + 1) * c

    def chunks_of(self, rank: int) -> Dict[int, Tuple[int, int]]:
        """{light: (k_begin, k_end)} of the shells of each group light held by rank."""
        j = self.group_index(rank)
        if j < 0:
            return {}
        p0, p1 = self.planes_of(rank)
        out = {}
        for q, l in enumerate(self.lights_of[j]):
            kb, ke = max(p0 - q * self.K, 0), min(p1 - q * self.K, self.K)
            out[l] = (kb, ke) if ke > kb else (0, 0)
        return out

    def split_lights(self, j: int) -> List[int]:
        """Lights of group j whose shells are held by more than one rank."""
        g = len(self.groups[j])
        if g == 1:
            return []
        c = len(self.lights_of[j]) * self.K // g
        return [l for q, l in enumerate(self.lights_of[j]) if (q * self.K) // c != ((q + 1) * self.K - 1) // c]


def lpt(costs: Sequence[float], bins: int) -> List[List[int]]:
    """Longest-processing-time-first assignment of items to `bins` bins."""
    order = sorted(range(len(costs)), key=lambda l: (-costs[l], l))
    load = [0.0] * bins
    out: List[List[int]] = [[] for _ in range(bins)]
    for l in order:
        r = min(range(bins), key=lambda q: (load[q], q))
        out[r].append(l)
        load[r] += costs[l]
    for x in out:
        x.sort()
    return out


def plan_layout(n_lights: int, world: int, K: int = 1, light_cost: Optional[Sequence[float]] = None,
                mode: str = "auto") -> Layout:
    """mode: "auto" ("light" if n_lights >= world else "shells"), "light",
    "shells" or "gaussian" (see the module docstring)."""
    if n_lights < 1 or world < 1:
        raise ValueError("need >= 1 light and >= 1 rank")
    if mode == "auto":
        mode = "light" if n_lights >= world else "shells"
    if mode == "light":
        if n_lights < world:
            raise ValueError(f"light-parallel needs >= {world} lights, got {n_lights}")
        cost = list(light_cost) if light_cost is not None else [1.0] * n_lights
        return Layout(world, [[r] for r in range(world)], lpt(cost, world), K, "light")
    if mode == "gaussian":
        if (n_lights * K) % world:
            raise ValueError(f"L*K = {n_lights * K} planes must divide over {world} ranks")
        return Layout(world, [list(range(world))], [list(range(n_lights))], K, "gaussian")
    if mode != "shells":
        raise ValueError(f"unknown layout {mode!r}")
    if n_lights >= world:
        return plan_layout(n_lights, world, K, light_cost, "light")
    g = world // n_lights
    extra = world - g * n_lights
    groups, r = [], 0
    for l in range(n_lights):
        size = g + (1 if l < extra else 0)
        if K % size:
            raise ValueError(f"K={K} must be divisible by the group size {size} for the shell reduce-scatter")
        groups.append(list(range(r, r + size)))
        r += size
    return Layout(world, groups, [[l] for l in range(n_lights)], K, "shells")


def shard_range(n: int, index: int, size: int) -> Tuple[int, int]:
    """Contiguous, balanced range of Gaussians for shard `index` of `size`."""
    base, rem = divmod(n, size)
    start = index * base + min(index, rem)
    return start, start + base + (1 if index < rem else 0)


def make_groups(layout: Layout) -> List[Optional[dist.ProcessGroup]]:
    """One process group per multi-rank light group (collective: every rank calls it)."""
    return [dist.new_group(ranks=g) if len(g) > 1 else None for g in layout.groups]


def _sub_lights(lights, ids):
    pos = np.asarray(lights["position"], np.float32).reshape(-1, 3)
    tm = np.asarray(lights["t_max"], np.float32).reshape(-1)
    return dict(position=pos[ids], t_max=tm[ids])


@dataclasses.dataclass
class ShardedAtlas:
    """What a rank holds after build_sharded: planes [p0, p1) of its group's
    flattened (light, shell) axis as T (data [p1 - p0, H, W]), i.e. per light
    the shell chunk chunks()[l] = (k_begin, k_end, view)."""
    lights: List[int]
    K: int
    p0: int
    p1: int
    data: Optional[torch.Tensor]

    def chunks(self) -> Dict[int, Tuple[int, int, Optional[torch.Tensor]]]:
        out = {}
        for q, l in enumerate(self.lights):
            kb, ke = max(self.p0 - q * self.K, 0), min(self.p1 - q * self.K, self.K)
            if ke > kb:
                a = q * self.K + kb - self.p0
                out[l] = (kb, ke, self.data[a:a + (ke - kb)])
        return out


BuildFn = Callable[..., torch.Tensor]


class ShardedBuilder:
    """The per-frame multi-GPU build of one rank (a7).  build_fn(gaussians,
    lights_subset, output_tau) -> [L', K, H, W] runs the single-GPU build
    (dgsm_build on the GPU, the oracle in CPU tests); exp_fn(tau) -> T in place
    (dgsm_exp_epilogue).  Buffers are allocated once and reused every frame."""

    def __init__(self, layout: Layout, pgroups, lights, res: int, build_fn: BuildFn,
                 exp_fn: Callable[[torch.Tensor], torch.Tensor], device="cpu"):
        self.layout, self.pgroups, self.res = layout, pgroups, res
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.j = layout.group_index(self.rank)
        self.idx, self.g = layout.shard_of(self.rank)
        self.my_lights = layout.lights_of[self.j] if self.j >= 0 else []
        self.sub = _sub_lights(lights, self.my_lights) if self.my_lights else None
        self.build_fn, self.exp_fn = build_fn, exp_fn
        K = layout.K
        self.p0, self.p1 = layout.planes_of(self.rank)
        self.mine = None
        if self.g > 1:
            self.mine = torch.empty((self.p1 - self.p0, res, res), dtype=torch.float32, device=device)

    def __call__(self, gaussians: Dict[str, torch.Tensor]) -> ShardedAtlas:
        K = self.layout.K
        if not self.my_lights:
            return ShardedAtlas([], K, 0, 0, None)
        if self.g == 1:
            T = self.build_fn(gaussians, self.sub, False)
            return ShardedAtlas(self.my_lights, K, 0, len(self.my_lights) * K, T.reshape(-1, self.res, self.res))
        n = next(iter(gaussians.values())).shape[0]
        s0, s1 = shard_range(n, self.idx, self.g)
        shard = {k: v[s0:s1] for k, v in gaussians.items()}
        tau = self.build_fn(shard, self.sub, True)                      # partial optical depth [L', K, H, W]
        flat = tau.reshape(-1, self.res, self.res)
        dist.reduce_scatter_tensor(self.mine, flat, op=dist.ReduceOp.SUM, group=self.pgroups[self.j])
        self.exp_fn(self.mine)                                           # Eq.4 on the owned planes, in place
        return ShardedAtlas(self.my_lights, K, self.p0, self.p1, self.mine)


def build_sharded(gaussians, lights, res: int, K: int, layout: Layout, pgroups, build_fn: BuildFn,
                  exp_fn) -> ShardedAtlas:
    """One-shot ShardedBuilder (tests)."""
    dev = next(iter(gaussians.values())).device
    return ShardedBuilder(layout, pgroups, lights, res, build_fn, exp_fn, dev)(gaussians)


QueryChunksFn = Callable[..., Tuple[torch.Tensor, torch.Tensor]]


def query_sharded(sa: ShardedAtlas, lights, positions: torch.Tensor, layout: Layout, pgroups,
                  chunks_fn: QueryChunksFn, combine_fn: Callable[[torch.Tensor, torch.Tensor], torch.Tensor],
                  res: int) -> torch.Tensor:
    """T(x) = prod_l T_l(x) over all lights of all ranks.

    chunks_fn(chunk_list, lights_subset, positions) -> (T_complete [m], partial [n_split, m])
        (dgsm_query_chunks; chunk_list[i] = (k_begin, k_end, split, tensor))
    combine_fn(partial, T) -> T *= prod partial (dgsm_query_combine)."""
    rank = dist.get_rank() if dist.is_initialized() else 0
    j = layout.group_index(rank)
    m = positions.shape[0]
    dev = positions.device
    T = torch.ones(m, dtype=torch.float32, device=dev)
    if j >= 0:
        split = layout.split_lights(j)
        held = sa.chunks()
        ids = [l for l in layout.lights_of[j] if l in held or l in split]
        chunk_list = []
        for l in ids:
            kb, ke, t = held.get(l, (0, 0, None))
            chunk_list.append((kb, ke, l in split, t))
        if ids:
            Tc, part = chunks_fn(chunk_list, _sub_lights(lights, ids), positions)
            if part.shape[0]:
                # the shells of a split light are spread over the group: sum the shares
                dist.all_reduce(part, op=dist.ReduceOp.SUM, group=pgroups[j])
                if layout.groups[j][0] == rank:  # count each split light once
                    combine_fn(part, Tc)
            T = Tc
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(T, op=dist.ReduceOp.PRODUCT)
    return T


class StrongStep:
    """One frame of the strong-scaling step of a rank (bench.py --config 3/5 at
    N > 1): ShardedBuilder (build + reduce-scatter + exp) then query_sharded
    (chunk query + all-reduce SUM of split lights + all-reduce PRODUCT).
    The CPU tests run this same object with oracle functions over gloo."""

    def __init__(self, layout: Layout, pgroups, lights, res: int, build_fn: BuildFn, exp_fn,
                 chunks_fn: QueryChunksFn, combine_fn, device="cpu"):
        self.builder = ShardedBuilder(layout, pgroups, lights, res, build_fn, exp_fn, device)
        self.layout, self.pgroups, self.lights, self.res = layout, pgroups, lights, res
        self.chunks_fn, self.combine_fn = chunks_fn, combine_fn
        self.atlas: Optional[ShardedAtlas] = None

    def __call__(self, gaussians: Dict[str, torch.Tensor], positions: torch.Tensor) -> torch.Tensor:
        self.atlas = self.builder(gaussians)
        return query_sharded(self.atlas, self.lights, positions, self.layout, self.pgroups, self.chunks_fn,
                             self.combine_fn, self.res)


def light_costs(plan_key_ranges: Sequence[Tuple[int, int]]) -> List[float]:
    """LPT cost of each light: its key count P_l (the accumulation work is
    proportional to the (texel, listed Gaussian) pairs 64 P_l)."""
    return [float(e - b) for b, e in plan_key_ranges]


# ---------------------------------------------------------------- CUDA path
def cuda_build_fn(builder_cache: Dict, res: int, K: int, **kw):
    """build_fn over the CUDA library: dgsm_build (Builder: plan + run in one C
    call, workspace kept across frames) into a cached output buffer."""
    from . import dgsm

    def fn(gaussians, lights, output_tau):
        L = int(np.asarray(lights["position"]).reshape(-1, 3).shape[0])
        key = (L, bool(output_tau))
        if key not in builder_cache:
            dev = next(iter(gaussians.values())).device
            builder_cache[key] = (dgsm.Builder(lights, res, K, dgsm.Options(output_tau=output_tau, **kw), device=dev),
                                  torch.empty((L, K, res, res), dtype=torch.float32, device=dev))
        b, out = builder_cache[key]
        b(gaussians, out)
        return out
    return fn


def cuda_exp_fn(tau):
    from . import dgsm
    return dgsm.exp_epilogue(tau, out=tau)


def cuda_chunks_fn(res: int, K: int):
    from . import dgsm

    def fn(chunk_list, lights, positions):
        return dgsm.query_chunks(chunk_list, lights, positions, res, K)
    return fn


def cuda_combine_fn(partial, T):
    from . import dgsm
    return dgsm.query_combine(partial, T)
