"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same
seeded inputs.  Tolerances (R12, north_star "1e-5 relative"):
  |grad_gpu - grad_orc|_j <= 1e-5 ((A|x|)_j + |b_j|) + 1e-12
  |g_gpu - g_orc|         <= 1e-5 (|c|^T x + gamma/2 x^T D_v^2 x + |mu|^T (A x + |b|))
  |x_gpu - x_orc|         <= 2e-6 (x in [0, max(r, u)])
Layout (buckets, permutation, offsets, tiles) is compared bit for bit.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from oracle.dual import BOX, BOXCUT, SIMPLEX, Problem, apply_A, dual_eval, row_sqnorms  # noqa: E402
from oracle.layout import dest_labels, tile_plan  # noqa: E402
from paper_2603_04621_b200 import MatchingProblem  # noqa: E402
from synth.matching import GenConfig, Instance, generate  # noqa: E402

DEV = torch.device("cuda", 0)


def make(cfg, kind=SIMPLEX, r=1.0, u=1.0, v=None):
    inst = generate(cfg)
    gp = MatchingProblem.from_instance(inst, kind=kind, r=r, u=u, v=v)
    P = Problem.from_instance(inst, kind=kind, r=r, u=(np.inf if kind == SIMPLEX else u), v=v)
    return inst, gp, P


def rand_lambda(rng, n, scale):
    return (rng.exponential(scale, n) * (rng.random(n) < 0.8)).astype(np.float32)


def check_grad(gp, P, lam32, gamma, x_check=True):
    lam_t = torch.from_numpy(lam32).to(DEV)
    grad, obj = gp.dual_grad(lam_t, gamma)
    torch.cuda.synchronize()
    grad, obj = grad.cpu().numpy(), obj.cpu().numpy()
    lam = lam32.astype(np.float64)
    ev = dual_eval(P, lam, gamma)
    absAx = apply_A(P, np.abs(ev.x))
    tol = 1e-5 * (absAx + np.abs(P.b)) + 1e-12
    err = np.abs(grad - ev.grad)
    assert np.all(err <= tol), (np.max(err / tol), np.argmax(err / tol))
    gscale = float(np.abs(P.c) @ np.abs(ev.x)) + abs(ev.reg) + float(np.abs(lam) @ (absAx + np.abs(P.b)))
    assert abs(obj[0] - ev.g) <= 1e-5 * gscale + 1e-12, (obj[0], ev.g)
    assert abs(obj[1] - ev.cx) <= 1e-5 * (float(np.abs(P.c) @ np.abs(ev.x)) + 1e-12)
    assert abs(obj[2] - ev.reg) <= 1e-5 * abs(ev.reg) + 1e-12
    assert obj[3] == pytest.approx(np.count_nonzero(ev.x > 0), abs=max(3, 1e-3 * P.nnz))
    if x_check:
        x = gp.primal(lam_t, gamma)
        torch.cuda.synchronize()
        np.testing.assert_allclose(x.cpu().numpy(), ev.x, atol=2e-6, rtol=0)
    return ev


CASES = {
    # name: (GenConfig, kind, r, u)
    "poisson_simplex": (GenConfig(num_sources=3000, num_dests=400, nnz_per_source=100, seed=21), SIMPLEX, 1.0, 1.0),
    "tiny_simplex": (GenConfig(num_sources=1000, num_dests=50, nnz_per_source=10, seed=1), SIMPLEX, 1.0, 1.0),
    "powerlaw_simplex": (GenConfig(num_sources=2500, num_dests=20000, length_law="powerlaw", max_len=9000,
                                   powerlaw_alpha=1.6, seed=22), SIMPLEX, 1.0, 1.0),
    "boxcut_m2": (GenConfig(num_sources=2000, num_dests=300, nnz_per_source=60, num_families=2, seed=23),
                  BOXCUT, 3.0, 1.0),
    "boxcut_powerlaw": (GenConfig(num_sources=1500, num_dests=20000, length_law="powerlaw", max_len=6000,
                                  powerlaw_alpha=1.5, seed=24), BOXCUT, 4.0, 0.6),
    "box_m3": (GenConfig(num_sources=1500, num_dests=200, nnz_per_source=30, num_families=3, seed=25), BOX, 1.0, 0.5),
    "bigJ_lambda_hot": (GenConfig(num_sources=1500, num_dests=60000, nnz_per_source=40, seed=26),
                        SIMPLEX, 2.0, 1.0),
    "bigJ_hot_short_blocks": (GenConfig(num_sources=6000, num_dests=100000, length_law="powerlaw", max_len=300,
                                        powerlaw_alpha=2.0, seed=34), SIMPLEX, 1.0, 1.0),
    "bigJ_boxcut_m2": (GenConfig(num_sources=1500, num_dests=30000, nnz_per_source=50, num_families=2, seed=35),
                       BOXCUT, 3.0, 1.0),
    "paper_table_like": (GenConfig(num_sources=20000, num_dests=2000, nnz_per_source=10, seed=36), SIMPLEX, 1.0, 1.0),
}


@pytest.mark.parametrize("name", list(CASES))
def test_dual_grad_matches_oracle(name):
    cfg, kind, r, u = CASES[name]
    inst, gp, P = make(cfg, kind, r, u)
    rng = np.random.default_rng(hash(name) % 2**32)
    n = gp.n
    for gamma in (0.01, 0.16, 1.0):
        check_grad(gp, P, np.zeros(n, np.float32), gamma)
        check_grad(gp, P, rand_lambda(rng, n, 2.0 / max(1.0, np.sqrt(inst.nnz / inst.num_dests))), gamma)
    check_grad(gp, P, rand_lambda(rng, n, 50.0), 0.05)     # large duals: most x = 0
    gp.close()


def test_primal_scaling_matches_oracle():
    cfg = GenConfig(num_sources=2000, num_dests=300, nnz_per_source=80, seed=27)
    rng = np.random.default_rng(5)
    v = rng.uniform(0.3, 3.0, cfg.num_sources).astype(np.float32)
    for kind, r, u in ((SIMPLEX, 1.0, 1.0), (BOXCUT, 2.0, 0.7)):
        inst, gp, P = make(cfg, kind, r, u, v=v)
        for gamma in (0.02, 0.3):
            check_grad(gp, P, rand_lambda(rng, gp.n, 0.1), gamma)
        gp.close()


def test_layout_bit_exact():
    cfg = GenConfig(num_sources=4000, num_dests=20000, length_law="powerlaw", max_len=9000, powerlaw_alpha=1.7,
                    seed=28)
    inst = generate(cfg)
    lens = np.diff(inst.row_ptr)
    lens[::37] = 0  # empty blocks
    rp = np.concatenate([[0], np.cumsum(lens)])
    keep = np.concatenate([np.arange(inst.row_ptr[i], inst.row_ptr[i] + lens[i]) for i in range(lens.size)])
    dest, c, a = inst.dest[keep], inst.c[keep], inst.a[:, keep]
    gp = MatchingProblem(rp, dest, a, c, inst.b, inst.num_dests)
    perm, off, tiles = gp.layout()
    operm, ooff, otiles, ototal = tile_plan(lens, gp.info["tile_cap"])
    np.testing.assert_array_equal(perm, operm)
    np.testing.assert_array_equal(off, ooff)
    np.testing.assert_array_equal(tiles, np.array(otiles).reshape(-1, 5))
    assert gp.info["nnz_layout"] == ototal
    ld, lc, la = gp.layout_data()
    for b in range(0, perm.size, 7):
        i = perm[b]
        sl = slice(rp[i], rp[i + 1])
        o = slice(off[b], off[b] + lens[i])
        np.testing.assert_array_equal(ld[o], dest[sl])
        np.testing.assert_array_equal(lc[o], c[sl])
        np.testing.assert_array_equal(la[:, o], a[:, sl])
    gp.close()


def test_row_sqnorms_match_oracle():
    cfg = GenConfig(num_sources=3000, num_dests=500, nnz_per_source=40, num_families=2, seed=29)
    inst, gp, P = make(cfg)
    got = gp.row_sqnorms()
    torch.cuda.synchronize()
    np.testing.assert_allclose(got.cpu().numpy(), row_sqnorms(P), rtol=1e-12, atol=0)
    gp.close()


def test_host_entry_equals_device_entry():
    cfg = GenConfig(num_sources=2000, num_dests=300, nnz_per_source=50, seed=30)
    inst, gp, P = make(cfg)
    lam = rand_lambda(np.random.default_rng(1), gp.n, 0.2)
    g_d, o_d = gp.dual_grad(torch.from_numpy(lam).to(DEV), 0.05)
    torch.cuda.synchronize()
    lam_h = torch.from_numpy(lam).pin_memory()
    g_h = torch.zeros(gp.n, dtype=torch.float64).pin_memory()
    o_h = torch.zeros(4, dtype=torch.float64).pin_memory()
    gp.dual_grad_host(lam_h, 0.05, g_h, o_h)
    np.testing.assert_allclose(g_h.numpy(), g_d.cpu().numpy(), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(o_h.numpy()[1:], o_d.cpu().numpy()[1:], rtol=1e-12)
    gp.close()


def test_edge_cases():
    # all blocks of length 1, J = 1, and an empty problem
    for cfg in (GenConfig(num_sources=500, num_dests=1, nnz_per_source=3, seed=31),
                GenConfig(num_sources=800, num_dests=3000, nnz_per_source=1.0, seed=32)):
        inst, gp, P = make(cfg)
        check_grad(gp, P, np.zeros(gp.n, np.float32), 0.1)
        check_grad(gp, P, rand_lambda(np.random.default_rng(2), gp.n, 1.0), 0.1)
        gp.close()
    gp = MatchingProblem(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros((1, 0), np.float32),
                         np.zeros(0, np.float32), np.ones(4, np.float32), 4)
    grad, obj = gp.dual_grad(torch.full((4,), 0.5, device=DEV), 0.1)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(grad.cpu().numpy(), -np.ones(4))
    assert obj.cpu().numpy()[0] == -2.0
    gp.close()


@pytest.mark.parametrize("kind,r,u", [(BOXCUT, 3.0, 1.0), (BOXCUT, 2.5, 0.5), (SIMPLEX, 1.0, 1.0)])
def test_near_flat_pieces(kind, r, u):
    """Blocks built so that the threshold equation F(phi) = sum clip(phi - d, 0, u) = r has a flat
    piece (or a kink) narrower than fp32 resolves: d_(K+1) - d_(K) = u (1 + delta), delta in
    [1e-7, 1e-3] (box-cut), resp. ties of the simplex threshold within 1e-7 relative.  The exact
    partition must be found (regression: an fp32 partition accepted as flat left x ~ 4e-5 on an
    entry the oracle sets to 0, sum x > r)."""
    rng = np.random.default_rng(33)
    I, L, gamma = 3000, 96, 0.01
    K = int(np.ceil(r / u)) if kind == BOXCUT else 1
    lens = np.full(I, L)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    J = 4000
    dest = np.concatenate([np.sort(rng.choice(J, L, replace=False)) for _ in range(I)]).astype(np.int32)
    base = rng.uniform(-8.0, -5.0, I)
    delta = 10.0 ** rng.uniform(-7, -3, I)
    c = np.empty(I * L)
    for i in range(I):
        off = np.sort(rng.uniform(0.0, 2.0, L))                      # the rest of the block, in s units
        off[:K] = np.sort(rng.uniform(0.0, 0.5 * u * gamma, K))        # K entries close to the minimum
        gap = (u if kind == BOXCUT else 0.0) * gamma * (1.0 + delta[i])
        off[K] = off[K - 1] + gap                                      # the (K+1)-th just past the flat piece
        off[K + 1:] = np.maximum(off[K + 1:], off[K] + 3 * gamma)
        c[rp[i]:rp[i + 1]] = base[i] + off[rng.permutation(L)]
    c = c.astype(np.float32)
    a = np.ones((1, I * L), np.float32)
    b = np.full(J, 10.0, np.float32)
    inst = Instance(I, J, 1, rp, dest, a, c, b)
    gp = MatchingProblem.from_instance(inst, kind=kind, r=r, u=u)
    P = Problem.from_instance(inst, kind=kind, r=r, u=(np.inf if kind == SIMPLEX else u))
    check_grad(gp, P, np.zeros(J, np.float32), gamma)
    gp.close()


@pytest.mark.parametrize("J,relabel", [(300, False), (60000, True), (100000, True)])
def test_dest_labels_rule(J, relabel):
    """Labels bit-exact against oracle.layout.dest_labels; the kernel sees labels, every output is
    in original coordinates (checked by the parity tests above on the same kinds of problems)."""
    inst = generate(GenConfig(num_sources=3000, num_dests=J, nnz_per_source=30, seed=60))
    gp = MatchingProblem.from_instance(inst)
    assert gp.info["relabeled"] == int(relabel)
    np.testing.assert_array_equal(gp.dest_labels(), np.array(dest_labels(inst.dest, J, relabel), np.int32))
    if relabel:
        assert 0 < gp.info["lambda_hot"] < J
    else:
        assert gp.info["lambda_hot"] == J and gp.info["lambda_in_smem"] == 1
    gp.close()


@pytest.mark.parametrize("J", [300, 60000])
def test_host_create_equals_device_create(J):
    """dl_problem_create_host (numpy input, streamed in source chunks) builds the same layout and
    the same gradient as dl_problem_create (CUDA tensors)."""
    inst = generate(GenConfig(num_sources=5000, num_dests=J, nnz_per_source=40, num_families=2, seed=61))
    v = np.random.default_rng(3).uniform(0.5, 2.0, inst.num_sources).astype(np.float32)
    gh = MatchingProblem(inst.row_ptr, inst.dest, inst.a, inst.c, inst.b, J, v=v)
    gd = MatchingProblem(*(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in
                           (inst.row_ptr, inst.dest, inst.a, inst.c, inst.b)), J, v=torch.from_numpy(v).cuda())
    for x, y in zip(gh.layout_data(), gd.layout_data()):
        np.testing.assert_array_equal(x, y)
    lam = torch.from_numpy(rand_lambda(np.random.default_rng(4), gh.n, 0.2)).to(DEV)
    g1, o1 = gh.dual_grad(lam, 0.05)
    g2, o2 = gd.dual_grad(lam, 0.05)
    torch.cuda.synchronize()
    np.testing.assert_allclose(g1.cpu().numpy(), g2.cpu().numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o1.cpu().numpy(), o2.cpu().numpy(), rtol=1e-12)
    gh.close()
    gd.close()


def test_standalone_calls_between_solver_steps():
    """dl_dual_grad / dl_primal between solver iterations use their own accumulator: solve(40) ->
    dual_grad -> primal -> solve(40) equals an uninterrupted solve(80)."""
    inst = generate(GenConfig(num_sources=4000, num_dests=300, nnz_per_source=50, seed=62))
    def run(interleave):
        gp = MatchingProblem.from_instance(inst)
        gp.agd_init(gamma0=0.05, use_jacobi=False)
        from paper_2603_04621_b200 import _lib as L
        if interleave:
            gp.solve(40)
            L.dl_agd_eval(gp.h)                     # a half-done iteration: accumulator full
            lam = torch.full((gp.n,), 0.3, device=DEV)
            gp.dual_grad(lam, 0.1)
            gp.primal(lam, 0.1)
            L.dl_dual_step(gp.h)
            gp.solve(39)
        else:
            gp.solve(80)
        h = gp.history()
        gp.close()
        return h
    a, b = run(True), run(False)
    assert a.size == b.size == 80
    np.testing.assert_allclose(a["g"], b["g"], rtol=1e-9)
