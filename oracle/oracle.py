"""Python side of the CPU ORACLE (arXiv:1811.05224).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module; the product package
paper_1811_05224_b200 never does.  Shares no code with the CUDA path.

Matrix entries come from the plain C oracle (stbem_oracle.c, ctypes).  This
module adds, in plain numpy and in the paper's order:
  * mass matrices M_h (primal, eq. 4) and M_h (dual pairing, Thm 1),
    the lumped dual mass (row sums);
  * the right-hand side (1/2 M_h + K_h) g of eq. (4), u0 = 0, dense or row by row
    (rhs_rows), and row-wise products of V_h, K_h, D_h (matvec_rows) for the full-size sampled tests
    (both pinned to the dense forms on C1);
  * full GMRES with modified Gram-Schmidt, x0 = 0, left preconditioning by
    C_V^{-1} = M_h^{-1} D_h M_h^{-T} (lumped or exact), stopping on the
    Givens estimate of the preconditioned relative residual;
  * the block forward substitution of the block-lower-triangular V_h;
  * the L2(Sigma) error of w_h against the exact Neumann datum;
  * the representation formula u = Vt w - W g at interior points (eq. 2; row f2, C code).
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstbem_oracle.so")
SRC_PATH = os.path.join(HERE, "stbem_oracle.c")


def build(force: bool = False) -> str:
    """compile the C oracle (gcc, OpenMP, no fast-math)"""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", LIB_PATH, SRC_PATH, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        d, i, p, ll = ctypes.c_double, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong
        for name in ("ora_e1", "ora_ein"):
            getattr(L, name).restype = d
            getattr(L, name).argtypes = [d]
        for name in ("ora_H", "ora_F", "ora_Q", "ora_ustar"):
            getattr(L, name).restype = d
            getattr(L, name).argtypes = [d, d, d]
        L.ora_ustar_dny.restype = d
        L.ora_ustar_dny.argtypes = [d, d, d, d]
        L.ora_mesh_new.restype = p
        L.ora_mesh_new.argtypes = [i, p, p, i, p, d]
        L.ora_mesh_free.argtypes = [p]
        L.ora_set_orders.argtypes = [p, i, i, i, i]
        L.ora_mesh_ng.restype = i
        L.ora_mesh_ng.argtypes = [p]
        L.ora_mesh_segments.argtypes = [p, p]
        for name in ("ora_entry_V", "ora_entry_K", "ora_entry_D"):
            getattr(L, name).restype = d
            getattr(L, name).argtypes = [p, i, i, i, i]
        L.ora_entries.argtypes = [p, i, ll, p, p, p]
        L.ora_dense.argtypes = [p, i, p]
        L.ora_dense_rows.argtypes = [p, i, ll, ll, p]
        L.ora_num_threads.restype = i
        L.ora_pair.restype = d
        L.ora_pair.argtypes = [p, i, i, i, i, i, i, d, d, d, d]
        L.ora_potential.argtypes = [p, p, p, ll, p, i, p]
        L.ora_initial_rhs.argtypes = [p, i, p, i, p, p, i, i, i, p]
        L.ora_potential_initial.argtypes = [p, i, p, i, p, p, ll, p, i, p]
        _lib = L
    return _lib


def e1(x):
    return lib().ora_e1(float(x))


KIND = {"V": 0, "K": 1, "D": 2}


class OracleMesh:
    """geometry + entry evaluation for one workload (workloads.Workload)"""

    def __init__(self, w, orders=None):
        self.w = w
        self._v = np.ascontiguousarray(w.vertices_flat(), dtype=np.float64)
        self._s = np.ascontiguousarray(w.segments_per_side, dtype=np.int32)
        self._t = np.ascontiguousarray(w.t_breaks, dtype=np.float64)
        self.h = lib().ora_mesh_new(len(w.vertices), self._v.ctypes.data, self._s.ctypes.data,
                                    w.n_steps, self._t.ctypes.data, float(w.alpha))
        if orders:
            lib().ora_set_orders(self.h, *orders)
        self.ng = w.n_gamma
        self.nt = w.n_steps
        self.n = self.ng * self.nt
        seg = np.zeros((self.ng, 8))
        lib().ora_mesh_segments(self.h, seg.ctypes.data)
        self.seg_a = seg[:, 0:2].copy()
        self.seg_b = seg[:, 2:4].copy()
        self.seg_h = seg[:, 4].copy()
        self.seg_n = seg[:, 5:7].copy()
        self.ht = np.diff(self._t)

    def __del__(self):
        try:
            lib().ora_mesh_free(self.h)
        except Exception:
            pass

    # -------------------------------------------------------------- matrices
    def entry(self, kind, a, i, b, j):
        f = {"V": lib().ora_entry_V, "K": lib().ora_entry_K, "D": lib().ora_entry_D}[kind]
        return f(self.h, int(a), int(i), int(b), int(j))

    def entries(self, kind, rows, cols):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty(len(rows))
        lib().ora_entries(self.h, KIND[kind], len(rows), rows.ctypes.data, cols.ctypes.data,
                          out.ctypes.data)
        return out

    def pair(self, ker, half, a, b, p, q, sx=(1.0, 1.0), sy=(1.0, 1.0)):
        """one segment-pair integral (ker 0=H, 1=F, 2=Q; half=1 for half segments)"""
        return lib().ora_pair(self.h, ker, half, a, b, p, q, sx[0], sx[1], sy[0], sy[1])

    def dense(self, kind):
        out = np.empty((self.n, self.n))
        lib().ora_dense(self.h, KIND[kind], out.ctypes.data)
        return out

    def dense_rows(self, kind, r0, nr):
        out = np.empty((nr, self.n))
        lib().ora_dense_rows(self.h, KIND[kind], int(r0), int(nr), out.ctypes.data)
        return out

    # ------------------------------------------------------ mass matrices (a6)
    def mass_primal(self):
        """M_h[(a,i),(a,n)] = <phi^10_(a,n), phi^0_(a,i)> = h_t(a) h_i / 2, n in {i, i+1}"""
        M = np.zeros((self.n, self.n))
        for a in range(self.nt):
            for i in range(self.ng):
                r = a * self.ng + i
                M[r, a * self.ng + i] += self.ht[a] * self.seg_h[i] / 2
                M[r, a * self.ng + (i + 1) % self.ng] += self.ht[a] * self.seg_h[i] / 2
        return M

    def mass_dual(self):
        """M_h[(a,l),(a,k)] = <phi^0_(a,k), psi_(a,l)> (Thm 1), dual hats of R6:
        int_{g_{l-1}} psi_l = h_{l-1} v-/4, int_{g_l} psi_l = h_l (2+v-+v+)/4, int_{g_{l+1}} psi_l = h_{l+1} v+/4"""
        ng = self.ng
        M = np.zeros((self.n, self.n))
        for a in range(self.nt):
            for l in range(ng):
                hm, h0, hp = self.seg_h[(l - 1) % ng], self.seg_h[l], self.seg_h[(l + 1) % ng]
                vm, vp = hm / (hm + h0), hp / (h0 + hp)
                r = a * ng + l
                M[r, a * ng + (l - 1) % ng] += self.ht[a] * hm * vm / 4
                M[r, a * ng + l] += self.ht[a] * h0 * (2 + vm + vp) / 4
                M[r, a * ng + (l + 1) % ng] += self.ht[a] * hp * vp / 4
        return M

    def dual_gram(self):
        """spatial Gram matrix G_Y[l, k] = int_Gamma psi_l psi_k of the dual hats (R6): on each half
        segment two hats are linear, int f g = L/6 (2 f0 g0 + f0 g1 + f1 g0 + 2 f1 g1)"""
        ng, h = self.ng, self.seg_h
        G = np.zeros((ng, ng))

        def add(l, k, L, f0, f1, g0, g1):
            v = L / 6.0 * (2 * f0 * g0 + f0 * g1 + f1 * g0 + 2 * f1 * g1)
            G[l % ng, k % ng] += v

        for i in range(ng):
            vm = h[(i - 1) % ng] / (h[(i - 1) % ng] + h[i])      # psi_i(x_i)
            vp = h[(i + 1) % ng] / (h[i] + h[(i + 1) % ng])      # psi_i(x_{i+1})
            L = h[i] / 2.0
            left = [(i, vm, 1.0), (i - 1, 1.0 - vm, 0.0)]        # [x_i, m_i]
            right = [(i, 1.0, vp), (i + 1, 0.0, 1.0 - vp)]       # [m_i, x_{i+1}]
            for half in (left, right):
                for (l, f0, f1) in half:
                    for (k, g0, g1) in half:
                        add(l, k, L, f0, f1, g0, g1)
        return G

    def stability_ratio(self):
        """the discrete inf-sup constant of the pairing <tau_h, v_h> between X^{0,0}(Sigma_h) and
        Y_h (eq. 5; SPEC's stability surrogate): the time factors h_t(a) and the H^{+-1/2, +-1/4}
        scalings cancel between the pairing and the two norms, leaving the spatial L^2 inf-sup
        sigma_min(G_Y^{-1/2} M_s G_X^{-1/2}) with M_s[l, k] = int psi_l phi_k (the dual mass of one
        step / h_t), G_X = diag(h_k), G_Y the dual-hat Gram matrix.  Returns (ratio, sigma_min(M_s))."""
        ng = self.ng
        Ms = self.mass_dual()[:ng, :ng] / self.ht[0]
        gx = 1.0 / np.sqrt(self.seg_h)
        wy, Uy = np.linalg.eigh(self.dual_gram())
        Gy = Uy @ np.diag(1.0 / np.sqrt(wy)) @ Uy.T
        B = Gy @ Ms @ np.diag(gx)
        return float(np.linalg.svd(B, compute_uv=False).min()), float(np.linalg.svd(Ms, compute_uv=False).min())

    def lumped_dual(self):
        """row sums of the dual mass: d_(a,l) = h_t(a)(h_{l-1} + 2 h_l + h_{l+1})/4"""
        return self.mass_dual().sum(axis=1)

    # ------------------------------------------------------------ rhs (a7)
    def rhs(self, K, g):
        """(1/2 M_h + K_h) g (eq. 4) with u0 = 0"""
        return 0.5 * self.mass_primal() @ g + K @ g

    def matvec_rows(self, kind, rows, x):
        """rows r = (a, i) of A x for A in {V_h, K_h, D_h}: sum over the causal columns (b <= a, P:86-88,
        P:104) of the C oracle's entries times x"""
        x = np.asarray(x, dtype=np.float64)
        out = np.empty(len(rows))
        for k, r in enumerate(rows):
            a = int(r) // self.ng
            cols = np.arange((a + 1) * self.ng)
            out[k] = float(self.entries(kind, np.full(len(cols), r), cols) @ x[cols])
        return out

    def rhs_rows(self, rows, g):
        """rows r = (a, i) of (1/2 M_h + K_h) g (eq. 4) without the dense matrices: K_h row
        entries (b <= a; causal) from the C oracle, the M_h row by P:89
        (h_t(a) h_i / 2 at columns (a, i) and (a, i + 1))"""
        g = np.asarray(g, dtype=np.float64)
        ng = self.ng
        out = np.empty(len(rows))
        for k, r in enumerate(rows):
            a, i = divmod(int(r), ng)
            cols = np.arange((a + 1) * ng)
            kg = float(self.entries("K", np.full(len(cols), r), cols) @ g[cols])
            mg = self.ht[a] * self.seg_h[i] / 2 * (g[a * ng + i] + g[a * ng + (i + 1) % ng])
            out[k] = 0.5 * mg + kg
        return out

    # ------------------------------------------------ representation formula (f2)
    def potential(self, w, g, pts, q=20):
        """u(x,t) = (Vt w)(x,t) - (W g)(x,t) at interior points pts[k] = (x1, x2, t), u0 = 0
        (eq. 2; time integrals exact, Gauss q per element: stbem_oracle.c)"""
        w = np.ascontiguousarray(w, dtype=np.float64)
        g = np.ascontiguousarray(g, dtype=np.float64)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(pts))
        lib().ora_potential(self.h, w.ctypes.data, g.ctypes.data, len(pts), pts.ctypes.data, int(q),
                            out.ctypes.data)
        return out

    def potential_initial(self, nodes, tris, u0, pts, q=8):
        """(M~_0 u0)(x,t) = int_Omega U*(x - y, t) u0_h(y) dy at points pts[k] = (x1, x2, t) (eq. 2,
        P:37-46): the initial-potential term of the representation formula (stbem_oracle.c)"""
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        tris = np.ascontiguousarray(tris, dtype=np.int32)
        u0 = np.ascontiguousarray(u0, dtype=np.float64)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(pts))
        lib().ora_potential_initial(self.h, len(nodes), nodes.ctypes.data, len(tris), tris.ctypes.data,
                                    u0.ctypes.data, len(pts), pts.ctypes.data, int(q), out.ctypes.data)
        return out

    # ------------------------------------------------ initial potential (f1)
    def initial_rhs(self, nodes, tris, u0, qx=4, qt_far=3, qt_near=8):
        """M_h^0 u0: u0 nodal on the triangulation (nodes (M,2), tris (T,3));
        exact time integrals, Gauss / collapsed-Gauss in space (stbem_oracle.c)"""
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        tris = np.ascontiguousarray(tris, dtype=np.int32)
        u0 = np.ascontiguousarray(u0, dtype=np.float64)
        out = np.empty(self.n)
        lib().ora_initial_rhs(self.h, len(nodes), nodes.ctypes.data, len(tris), tris.ctypes.data,
                              u0.ctypes.data, int(qx), int(qt_far), int(qt_near), out.ctypes.data)
        return out

    # ---------------------------------------------------------- L2 error
    def l2_error(self, wh, nq=10, exact=None):
        """|| w_h - w ||_{L2(Sigma)} and ||w||, Gauss nq x nq per element; exact(x, n, t) = d_n u
        (default: the BJ manufactured solution)"""
        from workloads.data import exact_neumann as bj_neumann
        exact_neumann = (lambda w_, x, n, t: exact(x, n, t)) if exact else bj_neumann
        xg, wg = np.polynomial.legendre.leggauss(nq)
        xg, wg = 0.5 * (xg + 1), 0.5 * wg
        t = self._t
        err2 = ref2 = 0.0
        W = wh.reshape(self.nt, self.ng)
        for a in range(self.nt):
            tt = t[a] + self.ht[a] * xg
            for i in range(self.ng):
                xx = self.seg_a[i][None, :] + xg[:, None] * (self.seg_b[i] - self.seg_a[i])[None, :]
                X = np.repeat(xx[:, None, :], nq, axis=1)
                TT = np.repeat(tt[None, :], nq, axis=0)
                ex = exact_neumann(self.w, X, self.seg_n[i][None, None, :], TT)
                ww = np.outer(wg, wg) * self.seg_h[i] * self.ht[a]
                err2 += np.sum(ww * (W[a, i] - ex) ** 2)
                ref2 += np.sum(ww * ex ** 2)
        return np.sqrt(err2), np.sqrt(ref2)


# --------------------------------------------------------------- solvers (a10)
def block_forward_solve(V, b, ng):
    """V is block lower triangular in time with N_Gamma x N_Gamma blocks"""
    n = len(b)
    nt = n // ng
    w = np.zeros(n)
    for a in range(nt):
        r = slice(a * ng, (a + 1) * ng)
        rhs = b[r] - V[r, : a * ng] @ w[: a * ng]
        w[r] = np.linalg.solve(V[r, r], rhs)
    return w


def make_preconditioner(mode, D=None, Mdual=None, lumped=None):
    """C_V^{-1} = M_h^{-1} D_h M_h^{-T}; mode 0 identity, 1 lumped, 2 exact"""
    if mode == 0:
        return lambda r: r.copy()
    if mode == 1:
        dinv = 1.0 / lumped
        return lambda r: dinv * (D @ (dinv * r))
    if mode == 2:
        return lambda r: np.linalg.solve(Mdual, D @ np.linalg.solve(Mdual.T, r))
    raise ValueError(mode)


def gmres(apply_A, apply_C, b, tol, max_iter=500):
    """full GMRES, modified Gram-Schmidt, x0 = 0, left preconditioning,
    stop when ||C(b - A x_k)|| / ||C b|| <= tol (Givens estimate)."""
    n = len(b)
    r0 = apply_C(b)
    beta = np.linalg.norm(r0)
    hist = [1.0]
    if beta == 0.0:
        return np.zeros(n), 0, hist
    Q = np.zeros((max_iter + 1, n))
    Hm = np.zeros((max_iter + 1, max_iter))
    cs = np.zeros(max_iter)
    sn = np.zeros(max_iter)
    gvec = np.zeros(max_iter + 1)
    gvec[0] = beta
    Q[0] = r0 / beta
    k = 0
    for k in range(max_iter):
        v = apply_C(apply_A(Q[k]))
        for j in range(k + 1):                  # modified Gram-Schmidt
            Hm[j, k] = np.dot(Q[j], v)
            v = v - Hm[j, k] * Q[j]
        Hm[k + 1, k] = np.linalg.norm(v)
        if Hm[k + 1, k] > 1e-300:
            Q[k + 1] = v / Hm[k + 1, k]
        for j in range(k):                      # previous Givens rotations
            t1 = cs[j] * Hm[j, k] + sn[j] * Hm[j + 1, k]
            Hm[j + 1, k] = -sn[j] * Hm[j, k] + cs[j] * Hm[j + 1, k]
            Hm[j, k] = t1
        den = np.hypot(Hm[k, k], Hm[k + 1, k])
        cs[k], sn[k] = Hm[k, k] / den, Hm[k + 1, k] / den
        Hm[k, k] = den
        Hm[k + 1, k] = 0.0
        gvec[k + 1] = -sn[k] * gvec[k]
        gvec[k] = cs[k] * gvec[k]
        hist.append(abs(gvec[k + 1]) / beta)
        if hist[-1] <= tol:
            break
    m = k + 1
    y = np.linalg.solve(np.triu(Hm[:m, :m]), gvec[:m])
    x = Q[:m].T @ y
    return x, m, hist
