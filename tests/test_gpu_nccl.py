"""The NCCL path on one GPU (A5): a one-rank communicator through dl_comm_unique_id /
dl_comm_init, the all-reduce of the m J + 4 accumulator captured inside the dl_solve graph.
With one rank the all-reduce is the identity, so the trajectory must equal the communicator-free
solve up to the summation order of the fused kernel's fp64 atomics (run-to-run, ~1e-15 relative).  (Multi-rank sharding is covered on CPU by tests/test_distributed_gloo.py;
this image gives one GPU per call.)"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2603_04621_b200 import MatchingProblem  # noqa: E402
from paper_2603_04621_b200 import _lib as L  # noqa: E402
from synth.matching import GenConfig, generate  # noqa: E402


def run(inst, with_comm):
    gp = MatchingProblem.from_instance(inst)
    if with_comm:
        L.dl_comm_init(gp.h, 0, 1, L.dl_comm_unique_id())
    rowsq = gp.row_sqnorms()
    gp.allreduce(rowsq)
    gp.set_jacobi(rowsq)
    gp.agd_init(gamma0=0.16, gamma_min=0.01, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5)
    gp.solve(120)
    h = gp.history()
    _, l2 = gp.dual()
    gp.close()
    return h, l2


def test_one_rank_nccl_solve_equals_local_solve():
    inst = generate(GenConfig(num_sources=20000, num_dests=500, nnz_per_source=30, seed=41))
    h0, l0 = run(inst, False)
    h1, l1 = run(inst, True)
    np.testing.assert_allclose(h1["g"], h0["g"], rtol=1e-12)
    np.testing.assert_allclose(l1, l0, rtol=1e-9, atol=1e-12 * np.abs(l0).max())
