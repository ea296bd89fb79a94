"""Multi-GPU min/max tournament: one process per GPU, torch.distributed.

Elements (each a batch of ciphertexts, u64[B][2][level][n]) are sharded contiguously: rank g owns
elements [g*T/G, (g+1)*T/G).  The tree is R20's fixed tree over element indices, so with T/G a
power of two the first log2(T/G) rounds pair elements inside one rank (run there as one
``bc_min_tree`` call) and every later round pairs the candidates of ranks g and g + 2^r': rank g
with g mod 2^(r'+1) = 2^r' sends its candidate to g - 2^r' (point-to-point send/recv over NCCL /
NVLink) and the receiver evaluates min(own, received) with its own candidate as `a` (the lower
element index).  The result therefore does not depend on G (bit-identical for G = 1, 2, 4, 8).
RNS limbs are never sharded; this exchange is the only collective on the path.

This module is host logic only: the compare/select arithmetic is done by ``ops`` (the CUDA
library through ``ProductOps``); the CPU tests drive the same logic with gloo and a stand-in.
"""
import torch
import torch.distributed as dist


class ProductOps:
    """tree / pair operations through libboostcom (every step in the CUDA kernels)."""

    def __init__(self, ctx, keys):
        self.ctx, self.keys = ctx, keys

    def tree(self, op, elems):
        return self.ctx.min_tree(self.keys, elems) if op == "min" else self.ctx.max_tree(self.keys, elems)

    def pair(self, op, a, b):
        return self.ctx.min(self.keys, a, b) if op == "min" else self.ctx.max(self.keys, a, b)

    def empty(self, shape):
        return torch.empty(shape, dtype=torch.int64, device=self.ctx.device)


def shard(T, world, rank):
    """element range [lo, hi) of `rank`; T/G must be a power of two so local rounds are the
    global tree's first rounds."""
    if T % world:
        raise ValueError("T = %d elements not divisible by %d ranks" % (T, world))
    per = T // world
    if world > 1 and per & (per - 1):
        raise ValueError("T / G = %d must be a power of two" % per)
    return rank * per, (rank + 1) * per


def cross_schedule(world):
    """[(r, role, peer)] per rank: the rank-level rounds of the fixed tree.  role 'send' (then
    the rank is done), 'recv' (combine), or absent (pass through)."""
    sched = {g: [] for g in range(world)}
    r = 1
    while r < world:
        for g in range(world):
            if g % (2 * r) == r:
                sched[g].append((r, "send", g - r))
            elif g % (2 * r) == 0 and g + r < world:
                sched[g].append((r, "recv", g + r))
        r *= 2
    return sched


def tournament(ops, local_elems, op, group=None):
    """Run the distributed tournament; returns the result on rank 0, None elsewhere."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    cand = ops.tree(op, local_elems) if len(local_elems) > 1 else local_elems[0]
    for r, role, peer in cross_schedule(world)[rank]:
        if role == "send":
            hdr = torch.tensor(list(cand.shape), dtype=torch.int64, device=cand.device)
            dist.send(hdr, peer, group=group)
            dist.send(cand.contiguous(), peer, group=group)
            return None
        hdr = torch.empty(4, dtype=torch.int64, device=cand.device)
        dist.recv(hdr, peer, group=group)
        other = ops.empty(tuple(int(x) for x in hdr.tolist()))
        dist.recv(other, peer, group=group)
        cand = ops.pair(op, cand, other)
    return cand if rank == 0 else None
