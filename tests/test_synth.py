"""The Appendix-B generator: determinism, shard equivalence and
statistics.  (Input construction only; no method arithmetic.)"""
import numpy as np

from synth.matching import GenConfig, capacities, dest_params, generate, generate_shard


def test_deterministic_and_shardable():
    cfg = GenConfig(num_sources=5000, num_dests=300, nnz_per_source=20, seed=7, chunk=1024)
    a = generate(cfg, threads=2)
    b = generate(cfg, threads=3)
    for f in ("row_ptr", "dest", "a", "c", "b"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    parts, load = [], 0
    for (s0, s1) in ((0, 1000), (1000, 2500), (2500, 5000)):
        sh, ld = generate_shard(cfg, s0, s1, threads=1)
        parts.append(sh)
        load = load + ld
        np.testing.assert_array_equal(sh.dest, a.dest[a.row_ptr[s0]:a.row_ptr[s1]])
        np.testing.assert_array_equal(sh.c, a.c[a.row_ptr[s0]:a.row_ptr[s1]])
    np.testing.assert_allclose(capacities(cfg, load), a.b, rtol=1e-6)


def test_structure_and_statistics():
    cfg = GenConfig(num_sources=40000, num_dests=500, nnz_per_source=12, seed=3, num_families=2)
    inst = generate(cfg)
    rp, d = inst.row_ptr, inst.dest
    lens = np.diff(rp)
    assert abs(lens.mean() - 12) < 0.5                     # Poisson(nu), few duplicates merged
    for i in range(0, 40000, 997):
        assert np.all(np.diff(d[rp[i]:rp[i + 1]]) > 0)   # dest strictly ascending per source
    assert np.all(inst.c <= 0) and np.all(-inst.c <= cfg.c_max + 1e-6)
    # family 0: a_ij / c_ij = -s_j constant per destination column
    dp = dest_params(cfg)
    ratio = inst.a[0] / (-inst.c.astype(np.float64))
    np.testing.assert_allclose(ratio, dp["s"][0][d], rtol=1e-6)
    # capacities: b/(l+eps) ~ U[0.5,1] -> mean 0.75
    p = dp["p"]
    expect_deg = 40000 * (1 - np.exp(-12 * p))             # P(j drawn >= once), N ~ Poisson(12)
    cnt = np.bincount(d, minlength=500)
    big = expect_deg > 200
    assert np.all(np.abs(cnt[big] - expect_deg[big]) < 5 * np.sqrt(expect_deg[big]))


def test_greedy_load_bruteforce():
    cfg = GenConfig(num_sources=300, num_dests=20, nnz_per_source=4, seed=9)
    inst = generate(cfg, threads=1)
    load = np.zeros(20)
    for i in range(300):
        sl = slice(inst.row_ptr[i], inst.row_ptr[i + 1])
        if sl.stop > sl.start:
            e = sl.start + int(np.argmax(inst.a[0][sl]))
            load[inst.dest[e]] += inst.a[0][e]
    np.testing.assert_allclose(inst.b, (dest_params(cfg)["rho"][0] * (load + cfg.slack_eps)).astype(np.float32),
                               rtol=1e-6)


def test_powerlaw_lengths():
    cfg = GenConfig(num_sources=20000, num_dests=20000, length_law="powerlaw", max_len=10000, seed=4)
    inst = generate(cfg)
    lens = np.diff(inst.row_ptr)
    assert lens.min() >= 1 and lens.max() > 1000
    frac1 = np.mean(lens == 1)
    assert 0.55 < frac1 < 0.66                              # P(1) = 1/zeta_10^4(2) ~ 0.608
