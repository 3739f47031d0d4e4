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
    (m x m) column-major tensor Z with Z[:, k] = eigenvector k.  Works on torch tensors.
    `gathered` is a list of P (max_shard x m) tensors or one (P * max_shard x m) tensor."""
    import torch
    if isinstance(gathered, (list, tuple)):
        gathered = torch.cat(list(gathered), 0)
    perm = torch.from_numpy(gather_perm(m, P, g)).to(gathered.device)
    return gathered.index_select(0, perm).t()          # row k = eigenvector k -> column-major Z


def gather_perm(m: int, P: int, g: int = 16) -> np.ndarray:
    """Row of the gathered (P * max_shard x m) array holding eigenvector k, for k = 0..m-1."""
    mc = max_shard(m, P, g)
    perm = np.empty(m, dtype=np.int64)
    for r in range(P):
        cols = shard_cols(m, P, r, g)
        perm[cols] = r * mc + np.arange(len(cols))
    return perm


def tri_layout(m: int, P: int, g: int = 16):
    """Triangular all-gather layout: rank r sends the rows 0..k of each of its eigenvectors k
    (column k is zero below row k), packed back to back.  Returns (per-rank (cols, heights,
    offsets) arrays, L = the longest rank's packed length), balanced by the serpentine map."""
    lay = []
    for r in range(P):
        c = shard_cols(m, P, r, g)
        h = c + 1
        off = np.concatenate([[0], np.cumsum(h)[:-1]]).astype(np.int64)
        lay.append((c, h.astype(np.int64), off))
    L = max(int(h.sum()) for _, h, _ in lay)
    return lay, L


def _pack(Zl, heights, offsets, out):
    if Zl.is_cuda:
        import paper_1607_01477_b200 as ms
        ms.pack_cols(Zl, heights, offsets, out)
    else:                                                     # CPU tensors (gloo tests)
        for q in range(heights.shape[0]):
            o, h = int(offsets[q]), int(heights[q])
            out[o:o + h] = Zl[:h, q]


def _unpack(inp, heights, offsets, dst, m, Z):
    if Z.is_cuda:
        import paper_1607_01477_b200 as ms
        ms.unpack_cols(inp, heights, offsets, dst, m, Z)
    else:
        for q in range(heights.shape[0]):
            o, h, k = int(offsets[q]), int(heights[q]), int(dst[q])
            Z[:h, k] = inp[o:o + h]
            Z[h:, k] = 0


def _panels(m: int, w: int):
    return [(c0, min(m, c0 + w)) for c0 in range(0, m, w)]


def block_panels(m: int, nb: int = 128):
    """Column panels of T in the order the blocked solve consumes them (op N, bottom-up: block b =
    rows [lo_b, hi_b) needs columns [lo_b, hi_b), rows 0 .. hi_b): [(lo_0, hi_0), (lo_1, hi_1), ...]
    from the right; the top block is the short one (R9).  The native path (trevc_*_dist) broadcasts T
    in exactly these panels and order."""
    out = []
    hi = m
    while hi > 0:
        lo = max(0, hi - nb)
        out.append((lo, hi))
        hi = lo
    return out


def pack_upper(T, m: int, w: int = 128):
    """The upper triangle of T as w-column panels T[0:c1, c0:c1] (rows up to the panel end, column
    by column) in one contiguous buffer: what the solve reads (the strictly lower triangle never
    is), ~m^2/2 elements instead of m^2."""
    import torch
    sizes = [c1 * (c1 - c0) for c0, c1 in _panels(m, w)]
    buf = torch.empty(sum(sizes), dtype=T.dtype, device=T.device)
    off = 0
    for (c0, c1), n in zip(_panels(m, w), sizes):
        buf[off:off + n].view(c1 - c0, c1).copy_(T[:c1, c0:c1].t())
        off += n
    return buf


def unpack_upper(buf, T, m: int, w: int = 128) -> None:
    off = 0
    for c0, c1 in _panels(m, w):
        n = c1 * (c1 - c0)
        T[:c1, c0:c1].copy_(buf[off:off + n].view(c1 - c0, c1).t())
        off += n


def broadcast_panels(T, m: int, *, rank: int, nb: int = 128, group=None):
    """T's upper triangle from rank 0 in block_panels order, one broadcast per panel, into T on the
    other ranks (the collective sequence of the native trevc_*_dist; there each panel's arrival
    gates its block of the solve)."""
    import torch
    import torch.distributed as dist
    for lo, hi in block_panels(m, nb):
        buf = torch.empty((hi - lo, hi), dtype=T.dtype, device=T.device)     # row q = column lo + q
        if rank == 0:
            buf.copy_(T[:hi, lo:hi].t())
        dist.broadcast(buf, src=0, group=group)
        if rank != 0:
            T[:hi, lo:hi].copy_(buf.t())


def trevc_sharded(T, m: int, solve_cols, *, rank: int, world: int, g: int = 16, group=None, nb: int = 128):
    """The multi-GPU TriangEig step, torch.distributed form of the native trevc_*_dist sequence:
    T's upper triangle from rank 0 panel by panel (block_panels order), this rank's block-cyclic
    column shard solved with `solve_cols`, a status all-reduce (max of the ranks' codes), the
    triangular shards (+ int32 exponents) all-gathered and unpacked on every rank.

    T: (m x m) tensor on every rank (contents only needed on rank 0; its upper triangle is
    overwritten elsewhere, the strictly lower triangle is not sent).
    solve_cols(T, cols, out) writes eigenvector cols[q] into column q of `out` (m x ncols,
    column-major) and returns the int32 exponents (ncols,).  Only rows 0..k of eigenvector k
    travel in the all-gather (tri_layout; the rest is zero by construction).
    The same collective calls run on NCCL (GPU) and gloo (CPU tests).
    Returns (Z (m x m, column-major), e (m,) int32), identical on every rank."""
    import torch
    import torch.distributed as dist
    if world > 1:
        broadcast_panels(T, m, rank=rank, nb=nb, group=group)
    cols = shard_cols(m, world, rank, g)
    if world == 1:
        send = torch.empty((len(cols), m), dtype=T.dtype, device=T.device)   # row q = eigenvector q
        el = solve_cols(T, cols, send.t())
        e = torch.empty(m, dtype=torch.int32, device=el.device)
        e[torch.from_numpy(cols).to(el.device)] = el
        return send.t(), e
    # this rank's shard, then only its upper-triangular part travels (≈ half the bytes)
    Zl = torch.empty((len(cols), m), dtype=T.dtype, device=T.device).t()   # m x ncols column-major
    status = 0
    try:
        el = solve_cols(T, cols, Zl)
    except Exception:                                                       # agree before the gather
        status, el = 1, torch.zeros(len(cols), dtype=torch.int32, device=T.device)
    st = torch.tensor([status], dtype=torch.int32, device=T.device)
    dist.all_reduce(st, op=dist.ReduceOp.MAX, group=group)
    if int(st.item()) != 0:
        raise RuntimeError("trevc_sharded: the shard solve failed on a rank")
    lay, L = tri_layout(m, world, g)
    dev = T.device
    _, h_r, off_r = lay[rank]
    send = torch.empty(L, dtype=T.dtype, device=dev)
    _pack(Zl, torch.from_numpy(h_r).to(dev), torch.from_numpy(off_r).to(dev), send)
    mc = max_shard(m, world, g)
    epad = torch.zeros(mc, dtype=torch.int32, device=el.device)
    epad[: len(cols)] = el
    out = torch.empty(world * L, dtype=send.dtype, device=dev)
    eout = torch.empty(world * mc, dtype=torch.int32, device=el.device)
    dist.all_gather_into_tensor(out, send, group=group)
    dist.all_gather_into_tensor(eout, epad, group=group)
    heights = np.concatenate([h for _, h, _ in lay])
    offsets = np.concatenate([off + r * L for r, (_, _, off) in enumerate(lay)])
    dst = np.concatenate([c for c, _, _ in lay]).astype(np.int64)
    Z = torch.empty((m, m), dtype=T.dtype, device=dev).t()
    _unpack(out, torch.from_numpy(heights).to(dev), torch.from_numpy(offsets).to(dev),
            torch.from_numpy(dst).to(dev), m, Z)
    perm = torch.from_numpy(gather_perm(m, world, g)).to(eout.device)
    e = eout.index_select(0, perm)
    return Z, e
