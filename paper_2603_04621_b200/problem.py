"""Owner of one dl_problem handle (marshalling only: every step runs in libdualip.so).

PyTorch is used for device memory, streams and process groups; nothing here
computes any part of the method.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L


class MatchingProblem:
    """One matching LP (or one rank's shard of sources) resident on a B200.

    Arrays follow include/dualip.h (source-major CSR; a family-major [m, nnz]).
    They may be numpy arrays (uploaded) or CUDA tensors; the library copies them
    into its own layout, so the caller's buffers can be dropped afterwards.
    """

    def __init__(self, row_ptr, dest, a, c, b, num_dests, kind=L.DL_PROJ_SIMPLEX, r=1.0, u=1.0, v=None,
                 device=0, stream=None):
        self.device = torch.device("cuda", device)
        dev = self.device
        # the library's work runs on this stream; methods order it against torch's current stream
        self.stream = stream if stream is not None else torch.cuda.Stream(device=dev)
        on_device = isinstance(dest, torch.Tensor) and dest.is_cuda
        if on_device:  # CUDA tensors: dl_problem_create reads them in place
            t = lambda x, dt: (x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))).to(
                dev, dt).contiguous()
        else:          # host arrays: dl_problem_create_host streams them into the layout (no device copy)
            t = lambda x, dt: np.ascontiguousarray(x.cpu().numpy() if isinstance(x, torch.Tensor) else x,
                                                   dtype=dt)
        i64, i32, f32 = ((torch.int64, torch.int32, torch.float32) if on_device else (np.int64, np.int32, np.float32))
        row_ptr = t(row_ptr, i64)
        dest = t(dest, i32)
        a = t(a, f32).reshape(-1)
        c = t(c, f32)
        b = t(b, f32)
        v = None if v is None else t(v, f32)
        n_el = (lambda x: x.numel()) if on_device else (lambda x: x.size)
        self.I = n_el(row_ptr) - 1
        self.J = int(num_dests)
        self.nnz = int(n_el(dest))
        self.m = n_el(a) // max(self.nnz, 1) if self.nnz else n_el(b) // self.J
        desc = L.dl_problem_desc(self.I, self.J, self.m, self.nnz, L.ptr(row_ptr), L.ptr(dest), L.ptr(a),
                                 L.ptr(c), L.ptr(b), L.ptr(v), int(kind), float(r), float(u), device,
                                 self.stream.cuda_stream)
        with torch.cuda.device(dev):
            if on_device:
                torch.cuda.current_stream(dev).synchronize()  # inputs written on torch's stream
                self.h = L.dl_problem_create(desc)
            else:
                self.h = L.dl_problem_create_host(desc)
        self.info = L.dl_problem_get_info(self.h)
        self.n = self.m * self.J

    @classmethod
    def from_instance(cls, inst, kind=L.DL_PROJ_SIMPLEX, r=1.0, u=1.0, v=None, device=0, stream=None):
        return cls(inst.row_ptr, inst.dest, inst.a, inst.c, inst.b, inst.num_dests, kind, r, u, v, device, stream)

    def _in(self):
        cur = torch.cuda.current_stream(self.device)
        if cur != self.stream:
            self.stream.wait_stream(cur)
        return cur

    def _out(self, cur):
        if cur != self.stream:
            cur.wait_stream(self.stream)

    # ---- A1 layout
    def layout(self):
        return L.dl_problem_layout(self.h, self.info["num_blocks"], self.info["num_tiles"])

    def layout_data(self):
        return L.dl_problem_layout_data(self.h, self.info["nnz_layout"], self.m)

    # ---- A2 preconditioning
    def row_sqnorms(self):
        out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        cur = self._in()
        L.dl_row_sqnorms(self.h, out)
        self._out(cur)
        return out

    def set_jacobi(self, row_sqnorm):
        cur = self._in()
        L.dl_set_jacobi(self.h, row_sqnorm)
        self._out(cur)

    # ---- A3 gradient
    def new_grad_buffers(self):
        return (torch.empty(self.n, dtype=torch.float64, device=self.device),
                torch.empty(4, dtype=torch.float64, device=self.device))

    def dual_grad(self, lam, gamma, out=None, flags=0):
        grad, obj = out if out is not None else self.new_grad_buffers()
        cur = self._in()
        L.dl_dual_grad(self.h, lam, gamma, grad, obj, flags)
        self._out(cur)
        return grad, obj

    def dual_grad_host(self, lam_host, gamma, grad_host, obj_host, flags=0):
        L.dl_dual_grad_host(self.h, lam_host, gamma, grad_host, obj_host, flags)
        return grad_host, obj_host

    def primal(self, lam, gamma):
        x = torch.empty(self.nnz, dtype=torch.float32, device=self.device)
        cur = self._in()
        L.dl_primal(self.h, lam, gamma, x)
        self._out(cur)
        return x

    # ---- A4/A5 solver
    def agd_init(self, **kw):
        L.dl_agd_init(self.h, **kw)

    def point(self):
        """The fp32 dual point mu_t the next evaluation uses (original coordinates)."""
        mu = np.zeros(self.n, np.float32)
        L.dl_agd_point(self.h, mu)
        return mu

    def dest_labels(self):
        return L.dl_problem_dest_labels(self.h, self.J)

    def solve(self, iters):
        L.dl_solve(self.h, iters)

    def history(self):
        return L.dl_agd_history(self.h)

    def dual(self):
        l1 = np.zeros(self.n)
        l2 = np.zeros(self.n)
        L.dl_agd_dual(self.h, l1, l2)
        return l1, l2

    def comm_init(self, rank, world, group=None):
        """NCCL communicator bootstrapped through torch.distributed (plumbing); world == 1
        without an initialised process group builds a one-rank communicator directly."""
        import torch.distributed as dist
        if world == 1 and not (dist.is_available() and dist.is_initialized()):
            L.dl_comm_init(self.h, 0, 1, L.dl_comm_unique_id())
        else:
            uid = L.dl_comm_unique_id() if rank == 0 else bytes(128)
            buf = torch.tensor(list(uid), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                buf = buf.to(self.device)
            dist.broadcast(buf, 0, group=group)
            L.dl_comm_init(self.h, rank, world, bytes(buf.cpu().tolist()))
        self.info = L.dl_problem_get_info(self.h)

    def allreduce(self, buf):
        cur = self._in()
        L.dl_comm_allreduce(self.h, buf, buf.numel())
        self._out(cur)

    def sync(self):
        L.dl_sync(self.h)

    def close(self):
        if getattr(self, "h", None) is not None:
            L.dl_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
