"""Thin ctypes binding of libstbem.so (include/stbem.h): argument marshalling only.

Every step of the path runs in the library's CUDA kernels.  There is no CPU fallback: if the
library cannot be loaded or no CUDA device is present, the calls raise.  Device vectors are
torch tensors (float64, on the mesh's CUDA device) passed by data_ptr(); streams are torch
streams (cuda_stream handle).
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libstbem.so")

BEM_OK, BEM_E_INVALID, BEM_E_NOMEM, BEM_E_CUDA, BEM_E_NCCL, BEM_E_NOT_CONVERGED, BEM_E_BREAKDOWN, BEM_E_STATE = range(8)
STATUS_NAMES = ["OK", "INVALID", "NOMEM", "CUDA", "NCCL", "NOT_CONVERGED", "BREAKDOWN", "STATE"]
MASS_PRIMAL, MASS_DUAL, MASS_DUAL_LUMPED = 0, 1, 2


class BemError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


class MeshDesc(ctypes.Structure):
    _fields_ = [("n_vertices", ctypes.c_int), ("vertices_xy", ctypes.POINTER(ctypes.c_double)),
                ("segments_per_side", ctypes.POINTER(ctypes.c_int)), ("n_steps", ctypes.c_int),
                ("t_breaks", ctypes.POINTER(ctypes.c_double)), ("alpha", ctypes.c_double),
                ("n_slices", ctypes.c_int)]


class MeshInfo(ctypes.Structure):
    _fields_ = [("n_gamma", ctypes.c_int), ("n_steps", ctypes.c_int), ("n", ctypes.c_longlong),
                ("n_slices", ctypes.c_int), ("n_owned_blocks", ctypes.c_int),
                ("entries_owned", ctypes.c_longlong), ("entries_total", ctypes.c_longlong),
                ("q_bulk", ctypes.c_int), ("kappa", ctypes.c_double), ("rank", ctypes.c_int),
                ("nranks", ctypes.c_int), ("local_rows", ctypes.c_longlong), ("local_row0", ctypes.c_longlong)]


class QuadOpts(ctypes.Structure):
    _fields_ = [("q_far", ctypes.c_int), ("q_near", ctypes.c_int), ("near_gap", ctypes.c_int),
                ("q_sing", ctypes.c_int), ("flags", ctypes.c_int)]


def quad_opts(q_bulk=0, q_sing=0, flags=0, q_near=0, near_gap=0):
    """bem_quad_opts; q_bulk is the order of the bulk time cells (the struct's q_far)"""
    return QuadOpts(int(q_bulk), int(q_near), int(near_gap), int(q_sing), int(flags))


class GmresOpts(ctypes.Structure):
    _fields_ = [("rel_tol", ctypes.c_double), ("max_iter", ctypes.c_int), ("precond", ctypes.c_int),
                ("flags", ctypes.c_int)]


class SolveReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("rel_residual", ctypes.c_double), ("true_rel_residual", ctypes.c_double),
                ("seconds_total", ctypes.c_double), ("seconds_matvec", ctypes.c_double),
                ("seconds_comm", ctypes.c_double), ("n_matvec_V", ctypes.c_int),
                ("n_matvec_D", ctypes.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


QUAD_LEGACY_SING = 1   # bem_quad_opts.flags: touching pairs by the per-lag singular kernel
QUAD_FULL_STORAGE = 2  # bem_quad_opts.flags: V_h / D_h stored full instead of symmetric packed
QUAD_KG_ENTRYWISE = 4  # bem_quad_opts.flags: fused K_h g pair by pair (no trial-moment table)


class AssemblyStats(ctypes.Structure):
    _fields_ = [("ms_bulk", ctypes.c_double), ("ms_near", ctypes.c_double), ("ms_sing", ctypes.c_double),
                ("evals_bulk", ctypes.c_longlong), ("evals_near", ctypes.c_longlong),
                ("q_bulk", ctypes.c_int), ("q_sing", ctypes.c_int), ("launches", ctypes.c_int),
                ("entries", ctypes.c_longlong), ("flops_bulk", ctypes.c_double),
                ("ms_records", ctypes.c_double), ("nodes_bulk", ctypes.c_longlong * 4),
                ("nodes_near", ctypes.c_longlong * 4), ("fused_sing", ctypes.c_int),
                ("nodes_bulk_tab", ctypes.c_longlong)]

    def as_dict(self):
        out = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            out[k] = list(v) if isinstance(v, ctypes.Array) else v
        return out


_lib = None
P = ctypes.c_void_p
PP = ctypes.POINTER(ctypes.c_void_p)
D = ctypes.c_double
I = ctypes.c_int
LL = ctypes.c_longlong

_SIGS = {
    "bem_version": (ctypes.c_char_p, []),
    "bem_last_error": (ctypes.c_char_p, []),
    "bem_launch_count": (LL, [I]),
    "bem_nccl_get_unique_id": (I, [P]),
    "bem_comm_create": (I, [P, I, I, I, PP]),
    "bem_comm_destroy": (None, [P]),
    "bem_comm_create_group": (I, [I, I, P]),
    "bem_comm_create_solo": (I, [I, I, I, PP]),
    "bem_plan_build": (I, [I, P]),
    "bem_plan_generator": (I, [I, P, P]),
    "bem_plan_owned_blocks": (I, [I, I, I, P, P]),
    "bem_slice_ranges": (I, [I, I, P]),
    "bem_mesh_create": (I, [ctypes.POINTER(MeshDesc), P, PP]),
    "bem_mesh_info_get": (I, [P, ctypes.POINTER(MeshInfo)]),
    "bem_mesh_destroy": (None, [P]),
    "bem_assemble_V": (I, [P, ctypes.POINTER(QuadOpts), P, PP]),
    "bem_assemble_K": (I, [P, ctypes.POINTER(QuadOpts), P, PP]),
    "bem_assemble_D": (I, [P, ctypes.POINTER(QuadOpts), P, PP]),
    "bem_assemble_M": (I, [P, I, P, PP]),
    "bem_matvec": (I, [P, D, P, D, P, P]),
    "bem_mass_solve": (I, [P, I, P, P, P]),
    "bem_rhs": (I, [P, P, P, P, P]),
    "bem_rhs_fused": (I, [P, P, P, P, P, P, P]),
    "bem_assemble_toeplitz": (I, [P, I, P, P, PP]),
    "bem_eval_potential": (I, [P, P, P, LL, P, P, P]),
    "bem_eval_potential_initial": (I, [P, I, P, I, P, P, LL, P, P, P]),
    "bem_rhs_initial": (I, [P, I, P, I, P, P, I, I, I, P, P]),
    "bem_solve_gmres": (I, [P, P, P, P, P, ctypes.POINTER(GmresOpts), ctypes.POINTER(SolveReport), P, P]),
    "bem_matrix_get": (I, [P, LL, LL, LL, LL, P]),
    "bem_matrix_get_entries": (I, [P, LL, P, P, P]),
    "bem_matrix_info": (I, [P, P, P, P]),
    "bem_matrix_stats": (I, [P, ctypes.POINTER(AssemblyStats)]),
    "bem_matrix_destroy": (None, [P]),
    "bem_release_storage": (I, []),
    "bem_eval_special": (I, [I, LL, P, P, P]),
    "bem_diag_fp64_rate": (I, [ctypes.c_double, P]),
}


def lib():
    """load libstbem.so (raises if it is missing: there is no fallback)"""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_1811_05224_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def symbols():
    return list(_SIGS)


def check(status):
    if status != BEM_OK:
        raise BemError(status, lib().bem_last_error().decode())
    return status


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _ptr(t):
    assert t.dtype.__str__() == "torch.float64" and t.is_cuda and t.is_contiguous(), "float64 contiguous CUDA tensor expected"
    return ctypes.c_void_p(t.data_ptr())


# ----------------------------------------------------------------------- plans (host)
def plan_build(P):
    out = np.zeros(P * P, dtype=np.int32)
    check(lib().bem_plan_build(P, out.ctypes.data))
    return out.reshape(P, P)


def plan_generator(P):
    out = np.zeros(P, dtype=np.int32)
    n = ctypes.c_int(0)
    check(lib().bem_plan_generator(P, out.ctypes.data, ctypes.addressof(n)))
    return out[: n.value].tolist()


def plan_owned_blocks(P, nranks, rank):
    out = np.zeros(P * (P + 1), dtype=np.int32)
    n = ctypes.c_int(0)
    check(lib().bem_plan_owned_blocks(P, nranks, rank, out.ctypes.data, ctypes.addressof(n)))
    return [tuple(x) for x in out[: 2 * n.value].reshape(-1, 2).tolist()]


def slice_ranges(n_steps, P):
    out = np.zeros(P + 1, dtype=np.int32)
    check(lib().bem_slice_ranges(n_steps, P, out.ctypes.data))
    return out.tolist()


def launch_count(reset=False):
    return lib().bem_launch_count(1 if reset else 0)


# ----------------------------------------------------------------------- comm
class Comm:
    """NCCL communicator; unique id exchanged through torch.distributed (caller's process group)"""

    def __init__(self, rank, world, device, unique_id=None):
        if unique_id is None:
            import torch.distributed as dist
            buf = [None]
            if rank == 0:
                uid = ctypes.create_string_buffer(128)
                check(lib().bem_nccl_get_unique_id(uid))
                buf = [bytes(uid.raw)]
            dist.broadcast_object_list(buf, src=0)
            unique_id = buf[0]
        uid = ctypes.create_string_buffer(unique_id, 128)
        h = ctypes.c_void_p()
        check(lib().bem_comm_create(uid, world, rank, device, ctypes.byref(h)))
        self.h = h
        self.rank, self.world = rank, world

    @classmethod
    def group(cls, world, device):
        """emulated ranks on one device (bem_comm_create_group): `world` handles, rank r driven by
        its own host thread"""
        hs = (ctypes.c_void_p * world)()
        check(lib().bem_comm_create_group(int(world), int(device), hs))
        out = []
        for r in range(world):
            c = cls.__new__(cls)
            c.h = ctypes.c_void_p(hs[r])
            c.rank, c.world = r, world
            out.append(c)
        return out

    @classmethod
    def solo(cls, world, rank, device):
        """rank `rank` of `world` alone on one device (bem_comm_create_solo): partial products only"""
        h = ctypes.c_void_p()
        check(lib().bem_comm_create_solo(int(world), int(rank), int(device), ctypes.byref(h)))
        c = cls.__new__(cls)
        c.h = h
        c.rank, c.world = rank, world
        return c

    def close(self):
        if self.h:
            lib().bem_comm_destroy(self.h)
            self.h = None


# ----------------------------------------------------------------------- mesh
class Mesh:
    def __init__(self, vertices, segments_per_side, t_breaks, alpha, n_slices=1, comm=None):
        self._v = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64).reshape(-1))
        self._s = np.ascontiguousarray(segments_per_side, dtype=np.int32)
        self._t = np.ascontiguousarray(t_breaks, dtype=np.float64)
        d = MeshDesc(len(self._v) // 2, self._v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                     self._s.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), len(self._t) - 1,
                     self._t.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(alpha), int(n_slices))
        h = ctypes.c_void_p()
        check(lib().bem_mesh_create(ctypes.byref(d), comm.h if comm else None, ctypes.byref(h)))
        self.h = h
        info = MeshInfo()
        check(lib().bem_mesh_info_get(self.h, ctypes.byref(info)))
        self.info = info
        self.ng, self.nt, self.n = info.n_gamma, info.n_steps, info.n

    @classmethod
    def from_workload(cls, w, n_slices=None, comm=None):
        return cls(w.vertices, w.segments_per_side, w.t_breaks, w.alpha,
                   n_slices if n_slices is not None else 1, comm)

    def close(self):
        if self.h:
            lib().bem_mesh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _assemble(self, fn, q_bulk=0, q_sing=0, legacy_sing=False, full_storage=False, q_near=0, near_gap=0,
                  stream=None):
        o = quad_opts(q_bulk, q_sing, (QUAD_LEGACY_SING if legacy_sing else 0) | (QUAD_FULL_STORAGE if full_storage else 0),
                      q_near, near_gap)
        h = ctypes.c_void_p()
        check(fn(self.h, ctypes.byref(o), _stream(stream), ctypes.byref(h)))
        return Matrix(h, self)

    def assemble_V(self, **kw):
        return self._assemble(lib().bem_assemble_V, **kw)

    def assemble_K(self, **kw):
        return self._assemble(lib().bem_assemble_K, **kw)

    def assemble_D(self, **kw):
        return self._assemble(lib().bem_assemble_D, **kw)

    def assemble_toeplitz(self, kind, q_bulk=0, q_sing=0, stream=None):
        """block-Toeplitz variant (uniform steps): kind 'V', 'K' or 'D' -> T_d = A(d, 0)"""
        o = quad_opts(q_bulk, q_sing)
        h = ctypes.c_void_p()
        check(lib().bem_assemble_toeplitz(self.h, "VKD".index(kind), ctypes.byref(o), _stream(stream), ctypes.byref(h)))
        return Matrix(h, self)

    def assemble_M(self, kind, stream=None):
        h = ctypes.c_void_p()
        check(lib().bem_assemble_M(self.h, int(kind), _stream(stream), ctypes.byref(h)))
        return Matrix(h, self)


class Matrix:
    def __init__(self, h, mesh):
        self.h = h
        self.mesh = mesh

    def close(self):
        if self.h:
            lib().bem_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        k, e, b = ctypes.c_int(), ctypes.c_longlong(), ctypes.c_longlong()
        check(lib().bem_matrix_info(self.h, ctypes.byref(k), ctypes.byref(e), ctypes.byref(b)))
        return {"kind": k.value, "entries": e.value, "bytes": b.value}

    def stats(self):
        st = AssemblyStats()
        check(lib().bem_matrix_stats(self.h, ctypes.byref(st)))
        return st.as_dict()

    def matvec(self, x, y, a=1.0, b=0.0, stream=None):
        check(lib().bem_matvec(self.h, float(a), _ptr(x), float(b), _ptr(y), _stream(stream)))
        return y

    def solve(self, x, y, transpose=False, stream=None):
        check(lib().bem_mass_solve(self.h, 1 if transpose else 0, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def get(self, r0, nr, c0, nc):
        out = np.empty((nr, nc))
        check(lib().bem_matrix_get(self.h, r0, nr, c0, nc, out.ctypes.data))
        return out

    def dense(self):
        n = self.mesh.n
        return self.get(0, n, 0, n)

    def entries(self, rows, cols):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty(len(rows))
        check(lib().bem_matrix_get_entries(self.h, len(rows), rows.ctypes.data, cols.ctypes.data, out.ctypes.data))
        return out


def rhs(K, Mp, g, b, stream=None):
    check(lib().bem_rhs(K.h, Mp.h, _ptr(g), _ptr(b), _stream(stream)))
    return b


def rhs_fused(mesh, Mp, g, b, q_bulk=0, q_sing=0, legacy_sing=False, stats=False, stream=None, entrywise=False):
    """b = 1/2 M g + K g with K_h computed on the fly and never stored (bem_rhs_fused); returns
    the K_h kernel statistics when stats=True (synchronises), else b.  entrywise: every regime-A
    node pair by pair (BEM_QUAD_KG_ENTRYWISE) instead of the trial-moment table"""
    o = quad_opts(q_bulk, q_sing, (QUAD_LEGACY_SING if legacy_sing else 0) | (QUAD_KG_ENTRYWISE if entrywise else 0))
    st = AssemblyStats() if stats else None
    check(lib().bem_rhs_fused(mesh.h, ctypes.byref(o), Mp.h, _ptr(g), _ptr(b),
                              ctypes.byref(st) if stats else None, _stream(stream)))
    return st.as_dict() if stats else b


def rhs_initial(mesh, nodes, tris, u0, b, qx=0, qt_far=0, qt_near=0, stream=None):
    """b <- b - M_h^0 u0 (bem_rhs_initial); nodes (M, 2) and tris (T, 3) host arrays, u0, b device"""
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    tris = np.ascontiguousarray(tris, dtype=np.int32)
    check(lib().bem_rhs_initial(mesh.h, len(nodes), nodes.ctypes.data, len(tris), tris.ctypes.data, _ptr(u0),
                                int(qx), int(qt_far), int(qt_near), _ptr(b), _stream(stream)))
    return b


def eval_potential(mesh, w, g, pts, out=None, stream=None):
    """u = Vt w - W g at interior points pts (npts x 3: x1, x2, t), u0 = 0 (bem_eval_potential)"""
    import torch
    pts = pts if isinstance(pts, torch.Tensor) else torch.tensor(pts, dtype=torch.float64, device=w.device)
    pts = pts.contiguous().reshape(-1, 3)
    out = out if out is not None else torch.empty(pts.shape[0], dtype=torch.float64, device=w.device)
    check(lib().bem_eval_potential(mesh.h, _ptr(w), _ptr(g), pts.shape[0], _ptr(pts), _ptr(out), _stream(stream)))
    return out


def eval_potential_initial(mesh, nodes, tris, u0, pts, out, stream=None):
    """out += (M~_0 u0)(x, t) at points pts (npts x 3: x1, x2, t > 0) (bem_eval_potential_initial);
    nodes (M, 2), tris (T, 3) host arrays, u0 nodal on the device"""
    import torch
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    tris = np.ascontiguousarray(tris, dtype=np.int32)
    pts = pts if isinstance(pts, torch.Tensor) else torch.tensor(pts, dtype=torch.float64, device=out.device)
    pts = pts.contiguous().reshape(-1, 3)
    check(lib().bem_eval_potential_initial(mesh.h, len(nodes), nodes.ctypes.data, len(tris), tris.ctypes.data,
                                           _ptr(u0), pts.shape[0], _ptr(pts), _ptr(out), _stream(stream)))
    return out


GMRES_FRESH_RESIDUAL = 1  # bem_gmres_opts.flags: true residual from fresh products


def solve_gmres(V, b, w, D=None, M=None, rel_tol=1e-10, max_iter=500, precond=0, history=True, stream=None,
                fresh_residual=False):
    o = GmresOpts(float(rel_tol), int(max_iter), int(precond), GMRES_FRESH_RESIDUAL if fresh_residual else 0)
    rep = SolveReport()
    hist = np.zeros(max_iter + 1) if history else None
    st = lib().bem_solve_gmres(V.h, D.h if D else None, M.h if M else None, _ptr(b), _ptr(w),
                               ctypes.byref(o), ctypes.byref(rep),
                               hist.ctypes.data if history else None, _stream(stream))
    if st not in (BEM_OK, BEM_E_NOT_CONVERGED, BEM_E_BREAKDOWN):
        check(st)
    r = rep.as_dict()
    r["status"] = STATUS_NAMES[st]
    if history:
        r["history"] = hist[: rep.iterations + 1].tolist()
    return r


def diag_fp64_rate(seconds=1.0):
    """live FP64 DFMA rate (TFLOP/s) of the current device over `seconds` (bem_diag_fp64_rate)"""
    out = ctypes.c_double(0.0)
    check(lib().bem_diag_fp64_rate(float(seconds), ctypes.addressof(out)))
    return out.value


def eval_special(which, x, out, stream=None):
    check(lib().bem_eval_special(int(which), x.numel(), _ptr(x), _ptr(out), _stream(stream)))
    return out
