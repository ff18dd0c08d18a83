"""ctypes binding of include/dualip.h (argument marshalling only).

Every function here has the name of the C entry point it calls and does nothing
but convert arguments (torch tensors / numpy arrays -> pointers) and raise
``DualipError`` on a non-zero dl_status.  All work runs in libdualip.so.  The
library is loaded at import; if it is missing the import fails loudly -- there
is no Python/CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DUALIP_LIB") or os.path.join(HERE, "lib", "libdualip.so")  # override: A/B diagnostics

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2603_04621_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

DL_PROJ_SIMPLEX, DL_PROJ_BOXCUT, DL_PROJ_BOX = 0, 1, 2
DL_GRAD_PARTIAL = 1
STATUS = {0: "DL_OK", 1: "DL_ERR_INVALID", 2: "DL_ERR_CUDA", 3: "DL_ERR_OOM", 4: "DL_ERR_STATE",
          5: "DL_ERR_NCCL", 6: "DL_ERR_UNSUPPORTED"}


class DualipError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class dl_problem_desc(C.Structure):
    _fields_ = [("num_sources", C.c_int64), ("num_dests", C.c_int32), ("num_families", C.c_int32),
                ("nnz", C.c_int64), ("row_ptr", C.c_void_p), ("dest", C.c_void_p), ("a", C.c_void_p),
                ("c", C.c_void_p), ("b", C.c_void_p), ("v", C.c_void_p), ("proj_kind", C.c_int32),
                ("proj_r", C.c_double), ("proj_u", C.c_double), ("device", C.c_int32), ("stream", C.c_void_p)]


class dl_problem_info(C.Structure):
    _fields_ = [("num_sources", C.c_int64), ("nnz", C.c_int64), ("nnz_layout", C.c_int64),
                ("num_blocks", C.c_int64), ("num_tiles", C.c_int64), ("num_big_tiles", C.c_int64),
                ("num_dests", C.c_int32), ("num_families", C.c_int32), ("tile_cap", C.c_int32),
                ("lambda_in_smem", C.c_int32), ("max_block_len", C.c_int32), ("num_buckets", C.c_int32),
                ("num_sms", C.c_int32), ("ctas", C.c_int32), ("device_bytes", C.c_int64),
                ("has_comm", C.c_int32), ("comm_rank", C.c_int32), ("comm_world", C.c_int32),
                ("relabeled", C.c_int32), ("lambda_hot", C.c_int32), ("pad_", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class dl_agd_params(C.Structure):
    _fields_ = [("gamma0", C.c_double), ("gamma_min", C.c_double), ("halve_every", C.c_int32),
                ("use_jacobi", C.c_int32), ("max_step", C.c_double), ("init_step", C.c_double),
                ("history_cap", C.c_int64)]


class dl_iter_record(C.Structure):
    _fields_ = [("iter", C.c_int64), ("g", C.c_double), ("gamma", C.c_double), ("eta", C.c_double),
                ("gnorm", C.c_double), ("infeas", C.c_double), ("nnz_x", C.c_double)]


HISTORY_DTYPE = np.dtype([("iter", "<i8"), ("g", "<f8"), ("gamma", "<f8"), ("eta", "<f8"),
                          ("gnorm", "<f8"), ("infeas", "<f8"), ("nnz_x", "<f8")])

_P = C.c_void_p
_sig = {
    "dl_abi_version": (C.c_int, []),
    "dl_last_error": (C.c_char_p, []),
    "dl_problem_create": (C.c_int, [C.POINTER(dl_problem_desc), C.POINTER(C.c_void_p)]),
    "dl_problem_create_host": (C.c_int, [C.POINTER(dl_problem_desc), C.POINTER(C.c_void_p)]),
    "dl_problem_dest_labels": (C.c_int, [_P, _P]),
    "dl_problem_destroy": (C.c_int, [_P]),
    "dl_problem_get_info": (C.c_int, [_P, C.POINTER(dl_problem_info)]),
    "dl_problem_layout": (C.c_int, [_P, _P, _P, _P]),
    "dl_problem_layout_data": (C.c_int, [_P, _P, _P, _P]),
    "dl_plan_tiles": (C.c_int, [_P, C.c_int64, C.c_int32, _P, _P, _P, _P, _P, _P]),
    "dl_plan_shards": (C.c_int, [_P, C.c_int64, C.c_int32, _P]),
    "dl_tile_cap": (C.c_int32, [C.c_int32, C.c_int32]),
    "dl_row_sqnorms": (C.c_int, [_P, _P]),
    "dl_set_jacobi": (C.c_int, [_P, _P]),
    "dl_dual_grad": (C.c_int, [_P, _P, C.c_double, _P, _P, C.c_uint32]),
    "dl_dual_grad_host": (C.c_int, [_P, _P, C.c_double, _P, _P, C.c_uint32]),
    "dl_primal": (C.c_int, [_P, _P, C.c_double, _P]),
    "dl_agd_init": (C.c_int, [_P, C.POINTER(dl_agd_params)]),
    "dl_agd_eval": (C.c_int, [_P]),
    "dl_agd_accumulator": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "dl_agd_gradient": (C.c_int, [_P, _P, _P]),
    "dl_dual_step": (C.c_int, [_P]),
    "dl_solve": (C.c_int, [_P, C.c_int64]),
    "dl_agd_point": (C.c_int, [_P, _P]),
    "dl_agd_history": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "dl_agd_dual": (C.c_int, [_P, _P, _P]),
    "dl_comm_unique_id": (C.c_int, [_P]),
    "dl_comm_init": (C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    "dl_comm_allreduce": (C.c_int, [_P, _P, C.c_int64]),
    "dl_debug_trace": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "dl_set_pass_events": (C.c_int, [_P, _P, _P]),
    "dl_sync": (C.c_int, [_P]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


def _ck(status):
    if status != 0:
        raise DualipError(status, _lib.dl_last_error().decode(errors="replace"))


def ptr(x):
    """Pointer of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    raise TypeError(type(x))


# ---- entry points, same names as the C ABI ------------------------------------
def dl_abi_version():
    return _lib.dl_abi_version()


def dl_last_error():
    return _lib.dl_last_error().decode(errors="replace")


def dl_problem_create(desc: dl_problem_desc):
    h = C.c_void_p()
    _ck(_lib.dl_problem_create(C.byref(desc), C.byref(h)))
    return h


def dl_problem_create_host(desc: dl_problem_desc):
    h = C.c_void_p()
    _ck(_lib.dl_problem_create_host(C.byref(desc), C.byref(h)))
    return h


def dl_problem_dest_labels(h, num_dests):
    lab = np.zeros(num_dests, np.int32)
    _ck(_lib.dl_problem_dest_labels(h, ptr(lab)))
    return lab


def dl_problem_destroy(h):
    _ck(_lib.dl_problem_destroy(h))


def dl_problem_get_info(h) -> dict:
    info = dl_problem_info()
    _ck(_lib.dl_problem_get_info(h, C.byref(info)))
    return info.as_dict()


def dl_problem_layout(h, num_blocks, num_tiles):
    perm = np.zeros(num_blocks, np.int64)
    off = np.zeros(num_blocks, np.int64)
    tiles = np.zeros((num_tiles, 5), np.int64)
    _ck(_lib.dl_problem_layout(h, ptr(perm), ptr(off), ptr(tiles)))
    return perm, off, tiles


def dl_problem_layout_data(h, nnz_layout, m):
    d = np.zeros(nnz_layout, np.int32)
    c = np.zeros(nnz_layout, np.float32)
    a = np.zeros((m, nnz_layout), np.float32)
    _ck(_lib.dl_problem_layout_data(h, ptr(d), ptr(c), ptr(a)))
    return d, c, a


def dl_plan_tiles(row_ptr: np.ndarray, tile_cap: int):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    I = rp.size - 1
    nb, nt, tot = C.c_int64(), C.c_int64(), C.c_int64()
    _ck(_lib.dl_plan_tiles(ptr(rp), I, tile_cap, None, None, None, C.byref(nb), C.byref(nt), C.byref(tot)))
    perm = np.zeros(nb.value, np.int64)
    off = np.zeros(nb.value, np.int64)
    tiles = np.zeros((nt.value, 5), np.int64)
    _ck(_lib.dl_plan_tiles(ptr(rp), I, tile_cap, ptr(perm), ptr(off), ptr(tiles), C.byref(nb), C.byref(nt),
                           C.byref(tot)))
    return perm, off, tiles, tot.value


def dl_plan_shards(row_ptr: np.ndarray, world: int):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.zeros(world + 1, np.int64)
    _ck(_lib.dl_plan_shards(ptr(rp), rp.size - 1, world, ptr(out)))
    return out


def dl_tile_cap(m, J):
    return _lib.dl_tile_cap(m, J)


def dl_row_sqnorms(h, out):
    _ck(_lib.dl_row_sqnorms(h, ptr(out)))


def dl_set_jacobi(h, row_sqnorm):
    _ck(_lib.dl_set_jacobi(h, ptr(row_sqnorm)))


def dl_dual_grad(h, lam, gamma, grad, obj, flags=0):
    _ck(_lib.dl_dual_grad(h, ptr(lam), float(gamma), ptr(grad), ptr(obj), flags))


def dl_dual_grad_host(h, lam, gamma, grad, obj, flags=0):
    _ck(_lib.dl_dual_grad_host(h, ptr(lam), float(gamma), ptr(grad), ptr(obj), flags))


def dl_primal(h, lam, gamma, x):
    _ck(_lib.dl_primal(h, ptr(lam), float(gamma), ptr(x)))


def dl_agd_init(h, gamma0, gamma_min=0.0, halve_every=25, use_jacobi=True, max_step=1e-3, init_step=1e-5,
                history_cap=0):
    prm = dl_agd_params(gamma0, gamma_min, halve_every, int(bool(use_jacobi)), max_step, init_step, history_cap)
    _ck(_lib.dl_agd_init(h, C.byref(prm)))


def dl_agd_eval(h):
    _ck(_lib.dl_agd_eval(h))


def dl_agd_accumulator(h):
    p, n = C.c_void_p(), C.c_int64()
    _ck(_lib.dl_agd_accumulator(h, C.byref(p), C.byref(n)))
    return p.value, n.value


def dl_agd_gradient(h, grad, obj):
    _ck(_lib.dl_agd_gradient(h, ptr(grad), ptr(obj)))


def dl_dual_step(h):
    _ck(_lib.dl_dual_step(h))


def dl_solve(h, iters):
    _ck(_lib.dl_solve(h, int(iters)))


def dl_agd_point(h, mu_out):
    _ck(_lib.dl_agd_point(h, ptr(mu_out)))


def dl_agd_history(h, cap=None):
    n = C.c_int64()
    _ck(_lib.dl_agd_history(h, None, 0, C.byref(n)))
    k = n.value if cap is None else min(cap, n.value)
    out = np.zeros(k, HISTORY_DTYPE)
    if k:
        _ck(_lib.dl_agd_history(h, ptr(out), k, C.byref(n)))
    return out


def dl_agd_dual(h, lam1_out=None, lam2_out=None):
    _ck(_lib.dl_agd_dual(h, ptr(lam1_out), ptr(lam2_out)))


def dl_comm_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _ck(_lib.dl_comm_unique_id(buf))
    return bytes(buf)


def dl_comm_init(h, rank, world, uid: bytes):
    buf = (C.c_char * 128).from_buffer_copy(uid)
    _ck(_lib.dl_comm_init(h, rank, world, buf))


def dl_comm_allreduce(h, buf, n):
    _ck(_lib.dl_comm_allreduce(h, ptr(buf), int(n)))


def dl_debug_trace(h):
    """Trace of the last fused pass (DUALIP_TRACE=1 at create): uint64, [ctas x 5] per-CTA records, then
    the completion time of every 4-tile chunk of the short-block phase."""
    n = C.c_int64()
    _ck(_lib.dl_debug_trace(h, None, 0, C.byref(n)))
    out = np.zeros(n.value, np.uint64)
    if n.value:
        _ck(_lib.dl_debug_trace(h, ptr(out), n.value, C.byref(n)))
    return out


def dl_set_pass_events(h, start=None, stop=None):
    """start/stop: torch.cuda.Event (timing enabled) or None; recorded around every fused launch."""
    _ck(_lib.dl_set_pass_events(h, C.c_void_p(start.cuda_event if start is not None else None),
                                C.c_void_p(stop.cuda_event if stop is not None else None)))


def dl_sync(h):
    _ck(_lib.dl_sync(h))
