"""Length bucketing, tile plan and shard plan (oracle, plain Python).

PAPER.md:367-369 ("Batched projection operator"): slices are grouped by length
into logarithmic buckets [2^(t-1), 2^t), so a block of length s >= 1 lies in
bucket t = floor(log2 s) + 1 and the number of buckets (GPU launches in the
paper) is at most 1 + floor(log2 s_max).

This framework keeps the buckets but, instead of padded dense slabs, lays the
blocks out bucket-contiguously in HBM and cuts each bucket into *tiles*
(reading R10):

* blocks of length 0 are skipped (PAPER.md silent; they carry no variables);
* blocks are ordered by (bucket descending, source id ascending);
* a bucket t >= BIG_BUCKET (length >= 256) block is a tile of its own, worked
  by a multi-warp group; smaller buckets are packed greedily, in that order,
  into tiles of at most ``tile_cap`` entries; a tile holding more than one
  round (``round_blocks(t, tile_cap)`` blocks) is trimmed to whole rounds, the trimmed
  blocks opening the next tile (no warp round runs with idle block groups);
* group widths: G lanes per block (1 for t <= 3, 2 for t = 4, 2^(t-4) for t = 5..8); with tiles
  of fewer than WIDE_CAP entries the widths of buckets 5..8 double, so that one round (32 / G
  blocks of a bucket's typical length) still fits one tile;
* every tile starts at an entry offset that is a multiple of 4 (16-byte TMA
  alignment); blocks inside a tile are contiguous; a block of bucket PAD_BUCKET <= t <
  BIG_BUCKET (16..255 entries) occupies its length rounded up to a multiple of 4 (padding
  entries follow it: 128-bit loads of whole 4-entry groups).

Shard plan ("balanced column split"): rank w of W owns the
contiguous sources [B_w, B_{w+1}) with B_w the first source whose CSR offset
reaches floor(w * nnz / W).
"""
from __future__ import annotations

import math

BIG_BUCKET = 9      # buckets >= 9 (length >= 256) are worked by multi-warp groups
PAD_BUCKET = 5      # buckets 5..8 store blocks padded to a multiple of ALIGN entries
ALIGN = 4           # entries (16 bytes of int32/float32)
WIDE_CAP = 384      # tiles below this many entries use doubled group widths in buckets 5..8


def bucket_of(s: int) -> int:
    """t = floor(log2 s) + 1, i.e. s in [2^(t-1), 2^t)."""
    if s < 1:
        raise ValueError("empty block has no bucket")
    return int(math.floor(math.log2(s))) + 1


def bucket_plan(lengths):
    """Paper's plan: {t: [block ids ascending]} and its launch count."""
    plan = {}
    for i, s in enumerate(lengths):
        if s > 0:
            plan.setdefault(bucket_of(int(s)), []).append(i)
    return dict(sorted(plan.items())), len(plan)


def group_lanes(t: int, tile_cap: int) -> int:
    """Lanes cooperating on one block of bucket t < BIG_BUCKET: 1 for t <= 3, 2 for t = 4, 2^(t-4)
    for t = 5..8 -- doubled (2^(t-3)) when tile_cap < WIDE_CAP."""
    if t <= 3:
        return 1
    if t == 4:
        return 2
    return 2 ** (t - 3) if tile_cap < WIDE_CAP else 2 ** (t - 4)


def round_blocks(t: int, tile_cap: int) -> int:
    """Blocks of bucket t < BIG_BUCKET one warp works at a time (a "round"): 32 / G with the
    group widths G of the fused kernel (group_lanes)."""
    return 32 // group_lanes(t, tile_cap)


def stored_len(s: int) -> int:
    """Entries a block of length s occupies in the layout (padded to ALIGN in buckets 5..8)."""
    t = bucket_of(s)
    return (s + ALIGN - 1) // ALIGN * ALIGN if PAD_BUCKET <= t < BIG_BUCKET else s


def tile_plan(lengths, tile_cap: int):
    """Returns (perm, blk_off, tiles, total) -- see module docstring.

    perm[b]    source id of the b-th block in layout order
    blk_off[b] entry offset of that block in the permuted arrays
    tiles      list of (first_block, num_blocks, entry_offset, num_entries, bucket)
    total      entries of the permuted arrays (including alignment gaps)
    """
    buckets, _ = bucket_plan(lengths)
    perm, blk_off, tiles = [], [], []
    off = 0
    for t in sorted(buckets, reverse=True):
        members = buckets[t]
        groups = []
        if t >= BIG_BUCKET:
            groups = [[i] for i in members]
        else:
            R = round_blocks(t, tile_cap)
            q = 0
            while q < len(members):
                n, tot = 0, 0
                while q + n < len(members) and (n == 0 or tot + stored_len(int(lengths[members[q + n]])) <= tile_cap):
                    tot += stored_len(int(lengths[members[q + n]]))
                    n += 1
                if n > R and q + n < len(members):   # trim to whole rounds (the bucket's last tile keeps all)
                    n -= n % R
                groups.append(members[q:q + n])
                q += n
        for grp in groups:
            off = (off + ALIGN - 1) // ALIGN * ALIGN
            start, b0 = off, len(perm)
            for i in grp:
                perm.append(i)
                blk_off.append(off)
                off += stored_len(int(lengths[i]))
            tiles.append((b0, len(grp), start, off - start, t))
    return perm, blk_off, tiles, off


def dest_labels(dest, num_dests: int, relabel: bool):
    """Destination labels of the layout (R15): when the duals do not all fit on chip,
    destinations are ordered by edge count, descending, ties by index ascending, and label l is
    the l-th of that order; otherwise the identity.  Returns lab[j]."""
    if not relabel:
        return list(range(num_dests))
    counts = [0] * num_dests
    for j in dest:
        counts[int(j)] += 1
    order = sorted(range(num_dests), key=lambda j: (-counts[j], j))
    lab = [0] * num_dests
    for l, j in enumerate(order):
        lab[j] = l
    return lab


def shard_bounds(row_ptr, world: int):
    """[B_0=0, B_1, ..., B_W=I] with B_w = min{i : row_ptr[i] >= floor(w*nnz/W)}."""
    I = len(row_ptr) - 1
    nnz = int(row_ptr[-1])
    out = [0]
    for w in range(1, world):
        target = (w * nnz) // world
        lo, hi = 0, I
        while lo < hi:                       # first i with row_ptr[i] >= target
            mid = (lo + hi) // 2
            if int(row_ptr[mid]) >= target:
                hi = mid
            else:
                lo = mid + 1
        out.append(max(lo, out[-1]))
    out.append(I)
    return out


__all__ = ["BIG_BUCKET", "PAD_BUCKET", "ALIGN", "WIDE_CAP", "bucket_of", "stored_len", "bucket_plan", "group_lanes", "round_blocks", "tile_plan",
           "dest_labels", "shard_bounds"]
