"""Pins for oracle.layout: the paper's bucket bracket and launch bound
(PAPER.md:369), the tile-plan invariants of DESIGN.md "HBM layout", and the
shard-plan balance."""
import math

import numpy as np

from oracle.layout import (ALIGN, BIG_BUCKET, PAD_BUCKET, WIDE_CAP, bucket_of, bucket_plan, group_lanes, round_blocks,
                           shard_bounds, stored_len,
                           tile_plan)


def test_bucket_bracket():
    for s in range(1, 5000):
        t = bucket_of(s)
        assert 2 ** (t - 1) <= s < 2 ** t


def test_paper_example_buckets():
    """lengths [1,2,3,5,8] -> {1}, {2,3}, {5}, {8}; 4 launches = 1 + floor(log2 8)."""
    plan, launches = bucket_plan([1, 2, 3, 5, 8])
    assert plan == {1: [0], 2: [1, 2], 3: [3], 4: [4]}
    assert launches == 4 == 1 + math.floor(math.log2(8))
    assert bucket_plan([1, 1, 1]) == ({1: [0, 1, 2]}, 1)
    assert bucket_plan([]) == ({}, 0)
    assert bucket_plan([0, 0, 3]) == ({2: [2]}, 1)       # empty blocks skipped


def test_launch_bound_and_padding_bound():
    rng = np.random.default_rng(0)
    for _ in range(200):
        lens = rng.integers(0, 3000, rng.integers(1, 300))
        plan, launches = bucket_plan(lens)
        if lens.max() > 0:
            assert launches <= 1 + math.floor(math.log2(lens.max()))
        for t, ids in plan.items():  # padded slab waste < 2x true entries
            assert len(ids) * (2 ** t - 1) < 2 * lens[ids].sum()


def test_round_blocks_match_group_widths():
    """round_blocks(t, cap) = 32 / G(t, cap): 32 one-lane groups for t <= 3, 16 two-lane groups for
    t = 4, then 2^(9-t) groups of 2^(t-4) lanes for t = 5..8 (tiles >= WIDE_CAP entries) or half
    as many groups of twice the width (smaller tiles); E G >= stored length of every block of the
    bucket with the kernel's slots per lane E (1, 3, 7 single-lane slots for t <= 3, 8 for t = 4;
    16 = four 4-entry groups for t >= 5, 8 in the wide mapping), and a round of blocks of the
    bucket's mean length (0.75 2^t) fits one tile."""
    for cap in (256, 380, WIDE_CAP, 460, 2048):
        wide = cap < WIDE_CAP
        E = {1: 1, 2: 3, 3: 7, 4: 8, 5: 16, 6: 16, 7: 16, 8: 16}
        if wide:
            E.update({5: 8, 6: 8, 7: 8, 8: 8})
        for t in range(1, BIG_BUCKET):
            G = group_lanes(t, cap)
            assert G * round_blocks(t, cap) == 32
            assert E[t] * G >= stored_len(2 ** t - 1)
            if t >= PAD_BUCKET:
                assert round_blocks(t, cap) * 0.75 * 2 ** t <= max(cap, 384)


def test_stored_len_padding():
    for s in range(1, 600):
        t = bucket_of(s)
        p = stored_len(s)
        if PAD_BUCKET <= t < BIG_BUCKET:
            assert p % ALIGN == 0 and s <= p < s + ALIGN and bucket_of(p) == t or (p == 2 ** t and s > 2 ** t - ALIGN)
        else:
            assert p == s


def test_tile_plan_invariants():
    rng = np.random.default_rng(1)
    for trial in range(60):
        n = int(rng.integers(1, 2000))
        if trial % 3 == 0:
            lens = np.minimum((rng.pareto(1.0, n) + 1).astype(int), 5000)
        else:
            lens = rng.poisson(rng.choice([3, 40, 120]), n)
        lens[rng.random(n) < 0.05] = 0
        cap = int(rng.choice([256, 424, 512, 1024]))
        perm, off, tiles, total = tile_plan(lens, cap)
        nz = np.flatnonzero(lens > 0)
        assert sorted(perm) == list(nz)                                # every nonempty block once
        keys = [(-bucket_of(int(lens[i])), i) for i in perm]
        assert keys == sorted(keys)                                    # (bucket desc, id asc)
        covered = 0
        for (b0, nb, toff, tn, t) in tiles:
            assert b0 == covered and nb >= 1
            covered += nb
            assert toff % ALIGN == 0
            members = perm[b0:b0 + nb]
            assert all(bucket_of(int(lens[i])) == t for i in members)
            assert off[b0] == toff
            for q in range(nb - 1):
                assert off[b0 + q + 1] == off[b0 + q] + stored_len(int(lens[members[q]]))
            assert tn == sum(stored_len(int(lens[i])) for i in members)
            if t >= BIG_BUCKET:
                assert nb == 1
            else:
                assert tn <= cap
        assert covered == len(perm)
        # greedy maximality, trimmed to whole warp rounds: a tile followed by one of the same bucket
        # holds the longest run from its first block that fits tile_cap, cut down to a multiple of
        # round_blocks(t, cap) when the run exceeds one round
        for (a, b) in zip(tiles, tiles[1:]):
            if a[4] == b[4] and a[4] < BIG_BUCKET:
                run, tot = 0, 0
                while a[0] + run < len(perm) and bucket_of(int(lens[perm[a[0] + run]])) == a[4] and \
                        (run == 0 or tot + stored_len(int(lens[perm[a[0] + run]])) <= cap):
                    tot += stored_len(int(lens[perm[a[0] + run]]))
                    run += 1
                R = round_blocks(a[4], cap)
                assert a[1] == (run if run <= R else run - run % R)
        assert total >= int(lens.sum())


def test_shard_bounds():
    rng = np.random.default_rng(2)
    for _ in range(100):
        lens = rng.integers(0, 200, rng.integers(1, 500))
        if rng.random() < 0.3:
            lens[rng.integers(0, lens.size)] = 10000
        rp = np.concatenate([[0], np.cumsum(lens)])
        for W in (1, 2, 3, 4, 8):
            B = shard_bounds(rp, W)
            assert B[0] == 0 and B[-1] == lens.size and all(x <= y for x, y in zip(B, B[1:]))
            nnz = rp[-1]
            for w in range(W):
                shard = rp[B[w + 1]] - rp[B[w]]
                assert shard <= math.ceil(nnz / W) + lens.max()
    assert shard_bounds(np.arange(0, 101, 1), 4) == [0, 25, 50, 75, 100]
