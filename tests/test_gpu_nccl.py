"""The NCCL path on one GPU (A5): a real one-rank communicator through dl_comm_unique_id /
dl_comm_init (has_comm is asserted), the all-reduce of the m J + 4 accumulator captured inside
the dl_solve graph, and the global relabelling dl_comm_init performs for problems whose duals do
not fit on chip.  With one rank the all-reduce is the identity, so the trajectory must equal the
communicator-free solve up to the summation order of the fused kernel's fp64 atomics (run to
run, ~1e-15 relative).  (Multi-rank sharding: tests/test_distributed_gloo.py on CPU; this image
gives one GPU per call.)"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2603_04621_b200 import MatchingProblem  # noqa: E402
from paper_2603_04621_b200 import _lib as L  # noqa: E402
from synth.matching import GenConfig, generate  # noqa: E402


def run(inst, with_comm, iters=120):
    gp = MatchingProblem.from_instance(inst)
    if with_comm:
        gp.comm_init(0, 1)
        assert gp.info["has_comm"] == 1 and gp.info["comm_world"] == 1
    else:
        assert gp.info["has_comm"] == 0
    rowsq = gp.row_sqnorms()
    gp.allreduce(rowsq)
    gp.set_jacobi(rowsq)
    gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
    gp.solve(iters)
    h = gp.history()
    _, l2 = gp.dual()
    lab = gp.dest_labels()
    gp.close()
    return h, l2, lab


@pytest.mark.parametrize("J", [500, 60000])
def test_one_rank_nccl_solve_equals_local_solve(J):
    inst = generate(GenConfig(num_sources=20000, num_dests=J, nnz_per_source=30, seed=41))
    h0, l0, lab0 = run(inst, False)
    h1, l1, lab1 = run(inst, True)
    np.testing.assert_array_equal(lab0, lab1)   # one rank: global counts == local counts
    np.testing.assert_allclose(h1["g"], h0["g"], rtol=1e-12)
    np.testing.assert_allclose(l1, l0, rtol=1e-9, atol=1e-12 * np.abs(l0).max())


def test_comm_reinit_replaces_communicator():
    inst = generate(GenConfig(num_sources=2000, num_dests=100, nnz_per_source=10, seed=42))
    gp = MatchingProblem.from_instance(inst)
    gp.comm_init(0, 1)
    gp.agd_init(gamma0=0.01)
    gp.solve(16)                                   # graph with the all-reduce captured
    gp.comm_init(0, 1)                             # replaced: old comm destroyed, graph dropped
    assert gp.info["has_comm"] == 1
    with pytest.raises(L.DualipError):
        gp.solve(8)                                # the AGD state was reset by dl_comm_init
    gp.agd_init(gamma0=0.01)
    gp.solve(16)
    assert gp.history().size == 16
    gp.close()
