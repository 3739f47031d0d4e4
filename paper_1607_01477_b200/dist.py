"""Multi-GPU sharding of the triangular-eigenvector driver (BASELINE north star).

Columns / shifts are independent units: every operation of Alg. 5 on column j touches only column j,
U and that column's scalars, so the eigenvectors shard across ranks with no exchange
during the solve.  The only collectives are the ones the north star names: a broadcast of T from
the root and an all-gather of the finished eigenvectors (+ their scale exponents).

Work balance: eigenvector k costs ~(k-1)^2 (the P:503-508 shortcut), so a contiguous split would
give the last rank ~1 - ((P-1)/P)^3 of the work; column groups of g are dealt block-cyclically in
serpentine order, which gives every rank ~1/P of the active columns at every block step.

This module is plumbing only (index maps, collectives, unpacking); the solve itself is whatever
`solve_cols(T, cols) -> (Z_local, exps_local)` the caller passes -- libmstrsm's trevc_*_cols on
the GPU path.  The host logic is exercised with the gloo backend on CPU in tests/test_dist.py.
"""
from __future__ import annotations

import numpy as np


def shard_rank(q, P: int):
    """Owner of column group q: serpentine block-cyclic order 0,1,..,P-1,P-1,..,1,0,0,1,..
    (plain cyclic order always hands the heaviest group of every round to rank P-1)."""
    q = np.asarray(q)
    c = q % P
    return np.where((q // P) % 2 == 0, c, P - 1 - c)


def shard_cols(m: int, P: int, r: int, g: int = 16) -> np.ndarray:
    """Eigenvector indices (ascending) owned by rank r of P: groups of g consecutive columns
    dealt to the ranks in serpentine block-cyclic order."""
    k = np.arange(m, dtype=np.int64)
    return k[shard_rank(k // g, P) == r]


def max_shard(m: int, P: int, g: int = 16) -> int:
    return max(len(shard_cols(m, P, r, g)) for r in range(P))


def unpack(gathered, m: int, P: int, g: int = 16):
    """gathered[r][q, :] = eigenvector shard_cols(m, P, r)[q] (rows padded to max_shard) ->
    (m x m) column-major tensor Z with Z[:, k] = eigenvector k.  Works on torch tensors."""
    import torch
    first = gathered[0]
    Z = torch.empty((m, m), dtype=first.dtype, device=first.device).t()   # column-major view
    for r in range(P):
        cols = torch.from_numpy(shard_cols(m, P, r, g)).to(first.device)
        Z[:, cols] = gathered[r][: len(cols)].t()
    return Z


def trevc_sharded(T, m: int, solve_cols, *, rank: int, world: int, g: int = 16, group=None):
    """Broadcast T from rank 0, solve this rank's block-cyclic column shard with `solve_cols`,
    all-gather the shards (vectors + int32 exponents) and unpack on every rank.

    T: (m x m) tensor on every rank (contents only needed on rank 0; overwritten elsewhere).
    solve_cols(T, cols) -> (Z_local (m x ncols, column q = eigenvector cols[q]), e_local (ncols,)).
    Returns (Z (m x m, column-major), e (m,) int32), identical on every rank."""
    import torch
    import torch.distributed as dist
    if world > 1:
        buf = T if T.is_contiguous() else T.t()          # column-major (m x m) views are .t() of a
        assert buf.is_contiguous()                       # contiguous buffer: send the storage
        dist.broadcast(buf, src=0, group=group)
    cols = shard_cols(m, world, rank, g)
    Zl, el = solve_cols(T, cols)
    if world == 1:
        e = torch.empty(m, dtype=torch.int32, device=el.device)
        e[torch.from_numpy(cols).to(el.device)] = el
        return Zl, e
    mc = max_shard(m, world, g)
    pad = torch.zeros((mc, m), dtype=Zl.dtype, device=Zl.device)           # row q = eigenvector q
    pad[: len(cols)] = Zl.t()
    epad = torch.zeros(mc, dtype=torch.int32, device=el.device)
    epad[: len(cols)] = el
    outs = [torch.empty_like(pad) for _ in range(world)]
    eouts = [torch.empty_like(epad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    dist.all_gather(eouts, epad, group=group)
    Z = unpack(outs, m, world, g)
    e = torch.empty(m, dtype=torch.int32, device=el.device)
    for r in range(world):
        c = torch.from_numpy(shard_cols(m, world, r, g)).to(el.device)
        e[c] = eouts[r][: len(c)]
    return Z, e
