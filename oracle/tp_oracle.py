"""TEST INFRASTRUCTURE ONLY -- numpy/scipy restatement of the reference hot path.

An independent CPU restatement of the reference algorithm (tpfem,
/root/reference/proj/include/tpfem) on the BASELINE grid physics.  It shares
no code with the product (paper_2502_21013_b200/) nor with the compiled
reference driver (oracle/_ref/libtpref.so); tests pin it against both:
  * against libtpref.so (the reference's own templates) on config 0,
  * against the reference's known-answer tests restated in
    tests/test_oracle_kats.py (symbols, monolithic all-at-once solve, DFT).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import it.

Function -> reference it restates:
  GridSetup             mesh.hpp:141-190 (uniform, no snapping), assembly.hpp:20-46
  GridSetup.mass_diag   assembly.hpp:50-65 (lumped, per-triangle sigma)
  GridSetup.loads       assembly.hpp:88-106, materials.hpp:60-65 (sum of sines)
  apply_k               assembly.hpp:126-140 (NonlinearOperator::apply)
  jacobian              assembly.hpp:153-177
  flux_jacobian_bounds  materials.hpp:112-128
  choose_nu_hat         assembly.hpp:236-303
  stiffness_frozen      assembly.hpp:68-84
  residual, block_l2    periodic.hpp:35-67
  symbol, periodic_solve periodic.hpp:146-198, 252-289
  newton_elliptic       solvers.hpp:131-182
  static_init           solvers.hpp:276-296
  stopping_check        solvers.hpp:100-103
  solve_m1_fixed_point  solvers.hpp:301-369
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

MASK64 = (1 << 64) - 1


class SolveError(RuntimeError):
    def __init__(self, msg, residual=-1.0):
        super().__init__(msg)
        self.residual = residual


def splitmix64_stream(seed: int, count: int) -> list[int]:
    out, state = [], seed & MASK64
    for _ in range(count):
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        out.append(z ^ (z >> 31))
    return out


def desc_to_dict(desc) -> dict:
    """Plain-python view of a tp_problem_desc (ctypes) or pass-through dict."""
    if isinstance(desc, dict):
        return desc
    mats = []
    for m in range(desc.n_materials):
        mt = desc.material[m]
        mats.append(dict(sigma=mt.sigma, sigma_noise=mt.sigma_noise, nu0=mt.nu0, nu_inf=mt.nu_inf,
                         bs=mt.bs, sources=[(mt.amp[h], mt.harmonic[h], mt.phase[h])
                                            for h in range(mt.n_harmonics)]))
    rects = [(r.x0, r.y0, r.x1, r.y1, r.material) for r in desc.rect[:desc.n_rects]]
    return dict(cells=desc.cells, steps=desc.steps, period=desc.period, materials=mats,
                rects=rects, noise_seed=desc.noise_seed, noise_lattice=desc.noise_lattice,
                noise_lo=desc.noise_lo, noise_hi=desc.noise_hi, noise_box=tuple(desc.noise_box),
                s_max=desc.s_max, flux_samples=desc.flux_samples)


class GridSetup:
    """Uniform P1 grid, materials, sigma, loads (BASELINE physics)."""

    def __init__(self, desc):
        d = desc_to_dict(desc)
        self.d = d
        c = self.c = int(d["cells"])
        self.N = int(d["steps"])
        self.T = float(d["period"])
        self.tau = self.T / self.N
        self.m = c - 1
        self.n = self.m * self.m
        h = 1.0 / c
        # cell material by centroid, painter's order (mesh.hpp:164-177)
        ii, jj = np.meshgrid(np.arange(c), np.arange(c), indexing="xy")  # [j, i]
        cx = (2.0 * ii + 1.0) / (2.0 * c)
        cy = (2.0 * jj + 1.0) / (2.0 * c)
        mat = np.zeros((c, c), dtype=np.int64)
        for (x0, y0, x1, y1, m) in d["rects"]:
            inside = (cx >= x0) & (cx <= x1) & (cy >= y0) & (cy <= y1)
            mat[inside] = m
        self.cell_mat = mat
        # triangles: t = 2*(j*c+i) + {0: (v00,v10,v11), 1: (v00,v11,v01)}
        nt = 2 * c * c
        self.tri_mat = np.repeat(mat.reshape(-1), 2)
        vid = lambda i, j: j * (c + 1) + i  # noqa: E731
        I = ii.reshape(-1)
        J = jj.reshape(-1)
        v00, v10, v01, v11 = vid(I, J), vid(I + 1, J), vid(I, J + 1), vid(I + 1, J + 1)
        tri = np.empty((nt, 3), dtype=np.int64)
        tri[0::2] = np.stack([v00, v10, v11], 1)
        tri[1::2] = np.stack([v00, v11, v01], 1)
        vx = (np.arange((c + 1) ** 2) % (c + 1)) / c
        vy = (np.arange((c + 1) ** 2) // (c + 1)) / c
        # dof numbering of interior vertices, row-major (mesh.hpp:92-102)
        vi = np.arange((c + 1) ** 2) % (c + 1)
        vj = np.arange((c + 1) ** 2) // (c + 1)
        interior = (vi > 0) & (vi < c) & (vj > 0) & (vj < c)
        dof_of = np.full((c + 1) ** 2, -1, dtype=np.int64)
        dof_of[interior] = (vj[interior] - 1) * self.m + (vi[interior] - 1)
        self.dof = dof_of[tri]
        # element geometry exactly as compute_element_data (assembly.hpp:28-46)
        p = [np.stack([vx[tri[:, k]], vy[tri[:, k]]], 1) for k in range(3)]
        area = 0.5 * ((p[1][:, 0] - p[0][:, 0]) * (p[2][:, 1] - p[0][:, 1])
                      - (p[2][:, 0] - p[0][:, 0]) * (p[1][:, 1] - p[0][:, 1]))
        inv2A = 1.0 / (2.0 * area)
        self.area = area
        self.gx = np.stack([(p[1][:, 1] - p[2][:, 1]) * inv2A, (p[2][:, 1] - p[0][:, 1]) * inv2A,
                            (p[0][:, 1] - p[1][:, 1]) * inv2A], 1)
        self.gy = np.stack([(p[2][:, 0] - p[1][:, 0]) * inv2A, (p[0][:, 0] - p[2][:, 0]) * inv2A,
                            (p[1][:, 0] - p[0][:, 0]) * inv2A], 1)
        # per-triangle sigma, seeded bilinear noise at triangle centroids
        mats = d["materials"]
        sig = np.array([mats[m]["sigma"] for m in range(len(mats))])[self.tri_mat]
        noisy = np.array([bool(mats[m]["sigma_noise"]) for m in range(len(mats))])[self.tri_mat]
        if noisy.any():
            lower = (np.arange(nt) % 2) == 0
            cell = np.arange(nt) // 2
            ci, cj = cell % c, cell // c
            tx = (3.0 * ci + np.where(lower, 2.0, 1.0)) / (3.0 * c)
            ty = (3.0 * cj + np.where(lower, 1.0, 2.0)) / (3.0 * c)
            sig = np.where(noisy, sig * self.noise(tx, ty), sig)
        self.sigma = sig
        self.nu0 = np.array([m["nu0"] for m in mats])
        self.nuinf = np.array([m["nu_inf"] for m in mats])
        self.bs = np.array([m["bs"] for m in mats])
        # scatter matrix: triangle-corner -> dof
        rows, cols = [], []
        for k in range(3):
            ok = self.dof[:, k] >= 0
            rows.append(self.dof[ok, k])
            cols.append(np.nonzero(ok)[0] * 3 + k)
        self.S = sp.csr_matrix((np.ones(sum(len(r) for r in rows)),
                                (np.concatenate(rows), np.concatenate(cols))),
                               shape=(self.n, 3 * nt))

    def noise(self, x, y):
        d = self.d
        L = int(d["noise_lattice"])
        vals = splitmix64_stream(int(d["noise_seed"]), L * L)
        lo, hi = d["noise_lo"], d["noise_hi"]
        v = np.array([lo + (hi - lo) * ((z >> 11) * 2.0 ** -53) for z in vals]).reshape(L, L)
        bx0, by0, bx1, by1 = d["noise_box"]

        def coord(p, a, b):
            s = np.clip((p - a) / (b - a) * (L - 1), 0.0, float(L - 1))
            i0 = np.minimum(np.floor(s).astype(np.int64), L - 2)
            return i0, s - i0

        a0, fx = coord(x, bx0, bx1)
        b0, fy = coord(y, by0, by1)
        val = ((1 - fx) * (1 - fy) * v[b0, a0] + fx * (1 - fy) * v[b0, a0 + 1]
               + (1 - fx) * fy * v[b0 + 1, a0] + fx * fy * v[b0 + 1, a0 + 1])
        return np.clip(val, lo, hi)

    # ---- material law (BASELINE) -------------------------------------
    def nu(self, mat, s):
        nu0, nuinf, bs = self.nu0[mat], self.nuinf[mat], self.bs[mat]
        s2 = s * s
        with np.errstate(invalid="ignore", divide="ignore"):
            v = nu0 + (nuinf - nu0) * s2 / (s2 + bs * bs)
        return np.where(nu0 == nuinf, nu0, v)

    def nu_prime(self, mat, s):
        nu0, nuinf, bs = self.nu0[mat], self.nuinf[mat], self.bs[mat]
        den = s * s + bs * bs
        with np.errstate(invalid="ignore", divide="ignore"):
            v = 2.0 * (nuinf - nu0) * s * bs * bs / (den * den)
        return np.where(nu0 == nuinf, 0.0, v)

    # ---- assembly -----------------------------------------------------
    def mass_diag(self):
        w = self.sigma * self.area / 3.0
        return self.S @ np.repeat(w, 3)

    def source_current(self, mat, t):
        out = 0.0
        for (amp, hrm, ph) in self.d["materials"][mat]["sources"]:
            out += amp * math.sin(2.0 * math.pi * hrm * t / self.T + ph)
        return out

    def loads(self):
        F = np.zeros((self.N, self.n))
        nmat = len(self.d["materials"])
        prof = []
        for m in range(nmat):
            w = np.where(self.tri_mat == m, self.area / 3.0, 0.0)
            prof.append(self.S @ np.repeat(w, 3))
        for i in range(self.N):
            t = (i + 1) * self.T / self.N
            for m in range(nmat):
                j = self.source_current(m, t)
                if j != 0.0:
                    F[i] += j * prof[m]
        return F

    def grads(self, U):
        """(gx, gy) per triangle for every slice: U (..., n) -> (..., nt)."""
        U = np.asarray(U)
        pad = np.concatenate([U, np.zeros(U.shape[:-1] + (1,))], -1)
        d = np.where(self.dof >= 0, self.dof, self.n)
        ux = pad[..., d]  # (..., nt, 3)
        gx = (ux * self.gx).sum(-1)
        gy = (ux * self.gy).sum(-1)
        return gx, gy

    def apply_k(self, U):
        gx, gy = self.grads(U)
        s = np.hypot(gx, gy)
        nu = self.nu(self.tri_mat, s)
        w = nu * self.area
        contrib = (w * gx)[..., None] * self.gx + (w * gy)[..., None] * self.gy
        flat = contrib.reshape(contrib.shape[:-2] + (-1,))
        return (self.S @ flat.reshape(-1, flat.shape[-1]).T).T.reshape(np.shape(U))

    def jacobian(self, u):
        gx, gy = self.grads(u)
        s = np.hypot(gx, gy)
        nu = self.nu(self.tri_mat, s)
        with np.errstate(invalid="ignore", divide="ignore"):
            rank1 = np.where(s > 0, self.nu_prime(self.tri_mat, s) / np.where(s > 0, s, 1), 0.0)
        rows, cols, vals = [], [], []
        for a in range(3):
            for b in range(3):
                ok = (self.dof[:, a] >= 0) & (self.dof[:, b] >= 0)
                iso = nu * (self.gx[:, a] * self.gx[:, b] + self.gy[:, a] * self.gy[:, b])
                da = gx * self.gx[:, a] + gy * self.gy[:, a]
                db = gx * self.gx[:, b] + gy * self.gy[:, b]
                rows.append(self.dof[ok, a])
                cols.append(self.dof[ok, b])
                vals.append((self.area * (iso + rank1 * da * db))[ok])
        return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(self.n, self.n))

    def stiffness_frozen(self, nu_hat):
        nu_hat = np.asarray(nu_hat, dtype=np.float64)
        if np.any(nu_hat <= 0):
            raise ValueError("frozen stiffness: nu_hat must be positive")
        coeff = nu_hat[self.tri_mat] * self.area
        rows, cols, vals = [], [], []
        for a in range(3):
            for b in range(3):
                ok = (self.dof[:, a] >= 0) & (self.dof[:, b] >= 0)
                rows.append(self.dof[ok, a])
                cols.append(self.dof[ok, b])
                vals.append((coeff * (self.gx[:, a] * self.gx[:, b]
                                      + self.gy[:, a] * self.gy[:, b]))[ok])
        return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(self.n, self.n))

    # ---- nu_hat -------------------------------------------------------
    def flux_jacobian_bounds(self, mat, s_lo, s_hi, samples):
        if not (s_lo >= 0) or not (s_hi >= s_lo):
            raise ValueError("flux bounds: need 0 <= s_lo <= s_hi")
        j = np.arange(samples)
        s = s_lo + (s_hi - s_lo) * j / (samples - 1)
        mt = np.full(samples, mat)
        nu = self.nu(mt, s)
        gp = nu + self.nu_prime(mt, s) * s
        return float(min(nu.min(), gp.min())), float(max(nu.max(), gp.max()))

    def choose_nu_hat(self, U0, mode="frozen_field", samples=2000):
        nmat = len(self.d["materials"])
        nu_hat = np.ones(5)
        q = 0.0
        if mode == "frozen_field":
            gx, gy = self.grads(U0)
            s = np.hypot(gx, gy)
        for r in range(nmat):
            lam_f, Lam_f = self.flux_jacobian_bounds(r, 0.0, self.d["s_max"], self.d["flux_samples"])
            if mode == "theory":
                nu_hat[r] = 0.5 * (lam_f + Lam_f)
                q = max(q, (Lam_f - lam_f) / (Lam_f + lam_f))
                continue
            sel = s[..., self.tri_mat == r]
            if sel.size == 0:
                nu_hat[r] = 0.5 * (lam_f + Lam_f)
                continue
            lo, hi = float(sel.min()), float(sel.max())
            margin = 0.2 * (hi - lo) + 1e-3
            lam, Lam = self.flux_jacobian_bounds(r, max(0.0, lo - margin), hi + margin, samples)
            nu_hat[r] = 0.5 * (lam + Lam)
            q = max(q, (Lam - lam) / (Lam + lam))
        return nu_hat, q


# ---- time-periodic block layer ---------------------------------------

def residual(g: GridSetup, U, F):
    """R = F - M(U - U_prev)/tau - K(U), U_prev periodic (periodic.hpp:35-58)."""
    m = g.mass_diag()
    Uprev = np.roll(U, 1, axis=0)
    return F - m[None, :] * ((U - Uprev) / g.tau) - g.apply_k(U)


def block_l2(R):
    return float(np.sqrt(np.sum(np.square(R))))


def symbol(k, N, tau):
    """Backward-difference circulant symbol (periodic.hpp:146-152)."""
    if k == 0:
        return 0.0 + 0.0j
    if 2 * k == N:
        return 2.0 / tau + 0.0j
    return (1.0 - complex(math.cos(-2.0 * math.pi * k / N), math.sin(-2.0 * math.pi * k / N))) / tau


class PeriodicSolver:
    """DFT along time + exact per-frequency sparse solves (periodic.hpp:126-301)."""

    def __init__(self, M, K_hat, tau, steps, imag_tol=1e-9, cache=True):
        self.M = sp.csr_matrix(M)
        self.K = sp.csr_matrix(K_hat)
        self.tau, self.N, self.imag_tol = tau, steps, imag_tol
        self.cache = {}
        self.use_cache = cache

    def _factor(self, k):
        if k in self.cache:
            return self.cache[k]
        lam = symbol(k, self.N, self.tau)
        A = (lam * self.M.astype(np.complex128) + self.K.astype(np.complex128)).tocsc()
        f = spla.splu(A)
        if self.use_cache:
            self.cache[k] = (f, A)
        return f, A

    def solve(self, G):
        N = self.N
        G = np.asarray(G, dtype=np.float64)
        W = np.fft.fft(G, axis=0)  # forward, unnormalised (fft.hpp:47,61-79)
        half = N // 2
        X = np.zeros_like(W)
        for k in range(half + 1):
            f, A = self._factor(k)
            b = W[k]
            if np.linalg.norm(b) == 0:
                x = np.zeros_like(b)
            else:
                x = f.solve(b)
                r = np.linalg.norm(A @ x - b) / np.linalg.norm(b)
                if not r <= 1e-10:
                    raise SolveError(f"sparse solve: relative residual {r} exceeds tolerance", r)
            X[k] = x
            if k != 0 and 2 * k != N:
                X[N - k] = np.conj(x)  # conjugate mirror (periodic.hpp:285-288)
        u = np.fft.ifft(X, axis=0)  # inverse divides by N (fft.hpp:48-51)
        re_n = float(np.sqrt(np.sum(u.real ** 2)))
        im_n = float(np.sqrt(np.sum(u.imag ** 2)))
        if im_n > self.imag_tol * max(re_n, 1e-300):
            raise SolveError(f"periodic solver: imaginary residue {im_n}", im_n / max(re_n, 1e-300))
        return u.real.copy()


def stopping_check(history, tol):
    if len(history) == 0:
        raise ValueError("stopping check: empty history")
    return history[-1] <= tol * history[0]


def newton_elliptic(g: GridSetup, rhs, u, rel_tol, max_newton, slope=1e-4, backtrack=0.5,
                    max_halvings=30):
    """Damped Newton for K(u) = rhs (mass_scale = 0) (solvers.hpp:131-182)."""
    def res(v):
        return rhs - g.apply_k(v)

    r = res(u)
    rnorm = float(np.linalg.norm(r))
    scale = max(float(np.linalg.norm(rhs)), rnorm)
    if scale == 0 or rnorm <= rel_tol * scale:
        return u, 0
    for step in range(1, max_newton + 1):
        J = g.jacobian(u).tocsc()
        delta = spla.spsolve(J, r)
        alpha, accepted = 1.0, False
        for _ in range(max_halvings + 1):
            trial = u + alpha * delta
            rt = res(trial)
            tn = float(np.linalg.norm(rt))
            if tn <= (1.0 - slope * alpha) * rnorm:
                u, r, rnorm, accepted = trial, rt, tn, True
                break
            alpha *= backtrack
        if not accepted:
            raise SolveError(f"newton: line search exhausted at residual {rnorm}", rnorm / scale)
        if rnorm <= rel_tol * scale:
            return u, step
    raise SolveError("newton: no convergence", rnorm / scale)


def static_init(g: GridSetup, F, static_tol=1e-8, max_newton=50):
    """Per-slice Newton from zero (solvers.hpp:276-296)."""
    U = np.zeros_like(F)
    counts = np.zeros(F.shape[0], dtype=np.int32)
    for i in range(F.shape[0]):
        try:
            U[i], counts[i] = newton_elliptic(g, F[i], np.zeros(g.n), static_tol, max_newton)
        except SolveError as e:
            raise SolveError(f"static init, step {i + 1}: {e}", e.residual) from e
    return U, counts


@dataclass
class M1Result:
    U: np.ndarray
    history: list = field(default_factory=list)
    contraction: list = field(default_factory=list)
    iterations: int = 0
    status: str = "converged"
    iterates: list | None = None


def solve_m1_fixed_point(g: GridSetup, K_hat, F, U0, tol=1e-4, max_outer=200, keep_iterates=False,
                         imag_tol=1e-9):
    """Fixed-point sweeps g = f + K_hat u - K(u), exact periodic solve (solvers.hpp:301-369)."""
    U = np.array(U0, dtype=np.float64, copy=True)
    res = M1Result(U=U, iterates=[U.copy()] if keep_iterates else None)
    res.history.append(block_l2(residual(g, U, F)))
    if not stopping_check(res.history, tol):
        solver = PeriodicSolver(sp.diags(g.mass_diag()), K_hat, g.tau, g.N, imag_tol=imag_tol)
        for k in range(1, max_outer + 1):
            G = F + (K_hat @ U.T).T - g.apply_k(U)
            U = solver.solve(G)
            res.iterations = k
            if keep_iterates:
                res.iterates.append(U.copy())
            res.history.append(block_l2(residual(g, U, F)))
            if stopping_check(res.history, tol):
                break
    res.status = "converged" if stopping_check(res.history, tol) else "max_iter"
    h = res.history
    res.contraction = [h[k + 1] / h[k] for k in range(len(h) - 1) if h[k] > 0]
    res.U = U
    return res
