"""Oracle: multilevel Newton iteration (Alg. 1), linear solves (Alg. 2), filtered line search.

Test infrastructure only (see oracle/__init__.py).

Passages followed:
* Alg. 1, §3.9: full-space gradient, Hessian, subspace direction,
  full-space correction, d = d_s + d_f, filtered backtracking line search, termination
  ||d_s|| / (h |V|) < eps.
* Alg. 2 L427-450 with readings R4 (exact coarse solves), R6 (right-hand side -g).
* §3.7.2: fixed-count Jacobi-PCG refinement from d_f = 0 (reading R5); NEXT-4 option:
  two-level PCG (Jacobi + SMS coarse correction) to a tolerance (reading N4, not in the paper).
* L616 and SPEC S:170-184: CCD (ground plane) and inversion filters with safety 0.9,
  backtracking by halving with strict decrease, alpha_min = 1e-8 (reading Q12).
* R3: one freshly assembled, fully integrated H for every stage (no cubature / lagging).
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import coarse, fem, ip

LS_SHRINK = 0.5
LS_MIN = 1e-8
FILTER_SAFETY = 0.9


def pcg(H, r, n_iter, Dinv=None):
    """Exactly n_iter Jacobi-PCG iterations on H d = r from d = 0, stop early only if rho == 0
    (P:477-484).  Returns d."""
    r = np.array(r, dtype=np.float64).ravel()
    if Dinv is None:
        Dinv = 1.0 / H.diagonal()
    d = np.zeros_like(r)
    z = Dinv * r
    p = z.copy()
    rho = r @ z
    for _ in range(n_iter):
        if rho == 0.0:
            break
        q = H @ p
        alpha = rho / (p @ q)
        d = d + alpha * p
        r = r - alpha * q
        z = Dinv * r
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new
    return d


def two_level_pcg(H, r, Us, S_chol, tol, ref_norm, max_iter, Dinv=None):
    """NEXT-4 (not in the paper -- reading N4 of DESIGN.md): PCG on H d = r from d = 0
    with the two-level preconditioner
        y = D^-1 v,   z = y + U_s S^-1 U_s^T (v - H y)
    (the Jacobi smoother of P:484, then the SMS coarse correction of Alg. 2 on the smoothed
    residual; S = U_s^T H U_s factorised once per Newton iteration; "A-DEF2" of Tang, Nabben, Vuik &
    Erlangga 2009, which equals the symmetric balancing preconditioner on residuals with
    U_s^T r = 0 -- what the SMS stage leaves: r1 = -g - H d_s), stopped at the first k with
    ||r_k||_2 <= tol ref_norm (ref_norm = ||g||_2) or k = max_iter.  Returns (d, iterations)."""
    r = np.array(r, dtype=np.float64).ravel()
    if Dinv is None:
        Dinv = 1.0 / H.diagonal()

    def precond(v):
        y = Dinv * v
        return y + Us @ coarse.cho_solve(S_chol, Us.T @ (v - H @ y))

    d = np.zeros_like(r)
    k = 0
    if np.linalg.norm(r) <= tol * ref_norm or max_iter <= 0:
        return d, 0
    z = precond(r)
    p = z.copy()
    rho = r @ z
    while True:
        q = H @ p
        alpha = rho / (p @ q)
        d = d + alpha * p
        r = r - alpha * q
        k += 1
        if np.linalg.norm(r) <= tol * ref_norm or k >= max_iter:
            return d, k
        z = precond(r)
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new


def block_jacobi_pcg(apply_S, b, blocks, tol, max_iter):
    """PCG on S q = b from q = 0 with the block-Jacobi preconditioner z = blockdiag(S_ii)^-1 r
    (12 x 12 blocks, one per handle: P:463-464) until ||r_k||_2 <= tol ||b||_2 ('a relative
    residual of 1e-4', reading C1 of DESIGN.md: unpreconditioned 2-norm, relative to the initial
    residual b) or max_iter iterations (NEXT-1).  apply_S(p) = S p (matrix-free,
    P:457-462); blocks: (n_handles, 12, 12).  Returns (q, iterations, ||r||_2 / ||b||_2)."""
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    q = np.zeros_like(b)
    if nb == 0.0:
        return q, 0, 0.0
    Linv = [np.linalg.inv(np.linalg.cholesky(B)) for B in blocks]   # S_ii^-1 = L^-T L^-1

    def precond(r):
        rr = r.reshape(-1, 12)
        return np.concatenate([Li.T @ (Li @ rr[k]) for k, Li in enumerate(Linv)])

    r = b.copy()
    z = precond(r)
    p = z.copy()
    rho = r @ z
    it = 0
    while it < max_iter and np.linalg.norm(r) > tol * nb:
        t = apply_S(p)
        alpha = rho / (p @ t)
        q = q + alpha * p
        r = r - alpha * t
        it += 1
        if np.linalg.norm(r) <= tol * nb:
            break
        z = precond(r)
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new
    return q, it, float(np.linalg.norm(r) / nb)


def galerkin_diagonal_blocks(U, H):
    """The 12 x 12 diagonal blocks (U_i^T H U_i) of the sandwich matrix, one per handle i
    (the block-Jacobi preconditioner of P:463-464), each by its definition."""
    H = H.tocsr()
    Uc = U.tocsc()
    nh = U.shape[1] // 12
    return np.array([(Uc[:, 12 * i:12 * i + 12].T @ (H @ Uc[:, 12 * i:12 * i + 12])).toarray() for i in range(nh)])


def subspace_direction(H, g, Ua, Us, coarse_mode="exact", tol=1e-4, max_iter=None):
    """Alg. 2 SolveSubspaceDirection with rhs -g (R6).  coarse_mode = "exact": Cholesky solves (R4);
    "pcg": the paper's solves: block-Jacobi PCG to relative residual tol on
    the matrix-free sandwich U^T H U p = U^T (H (U p)) (NEXT-1; max_iter caps the iterations,
    None = no cap).  In "pcg" mode S_a / S are not formed; the returned "matrices" are then the
    iteration counts (affine, SMS).

    Returns d_s, d_a and the coarse matrices S_a, S (exact) or the iteration counts (pcg)."""
    if coarse_mode == "pcg":
        g = g.ravel()
        H = H.tocsr()
        cap = np.iinfo(np.int64).max if max_iter is None else max_iter
        qa, ita, _ = block_jacobi_pcg(lambda p: Ua.T @ (H @ (Ua @ p)), Ua.T @ (-g),
                                      galerkin_diagonal_blocks(Ua, H), tol, cap)
        da = Ua @ qa
        r1 = -g - H @ da
        qs, its, _ = block_jacobi_pcg(lambda p: Us.T @ (H @ (Us @ p)), Us.T @ r1,
                                      galerkin_diagonal_blocks(Us, H), tol, cap)
        ds = da + Us @ qs
        return ds, da, ita, its
    g = g.ravel()
    Sa = coarse.galerkin(Ua, H)
    qa = coarse.cho_solve(coarse.cholesky(Sa), Ua.T @ (-g))
    da = Ua @ qa
    r1 = -g - H @ da
    S = coarse.galerkin(Us, H)
    qs = coarse.cho_solve(coarse.cholesky(S), Us.T @ r1)
    ds = da + Us @ qs
    return ds, da, Sa, S


def ccd_alpha(model, x, d):
    """Ground-plane CCD: alpha = min(1, 0.9 min_{v: n.d_v < 0} dist_v / (-n.d_v))."""
    if model.ground is None:
        return 1.0
    dist, nrm = ip.ground_distance(model, x)
    vel = d @ nrm
    f = model.free & (vel < 0.0)
    if not np.any(f):
        return 1.0
    return float(min(1.0, FILTER_SAFETY * np.min(dist[f] / (-vel[f]))))


def det_poly(A, B):
    """Coefficients (c0, c1, c2, c3) of det(A + t B) = c0 + c1 t + c2 t^2 + c3 t^3.

    Computed from the exact multilinearity of det in the columns: each coefficient is a sum
    of determinants with columns drawn from A or B."""
    cols = lambda M, k: M[..., :, k]
    c = [np.zeros(A.shape[:-2]) for _ in range(4)]
    for mask in range(8):
        pick = [(B if (mask >> k) & 1 else A) for k in range(3)]
        M = np.stack([cols(pick[k], k) for k in range(3)], axis=-1)
        c[bin(mask).count("1")] = c[bin(mask).count("1")] + np.linalg.det(M)
    return c


def smallest_positive_root(c):
    """Smallest real root t > 0 of c0 + c1 t + c2 t^2 + c3 t^3 (inf if none), per element:
    the eigenvalues of the companion matrix of the leading-nonzero polynomial (what
    numpy.roots computes), batched over the elements of each degree."""
    c0, c1, c2, c3 = [np.asarray(ci, dtype=np.float64).ravel() for ci in c]
    out = np.full(c0.shape, np.inf)
    deg = np.where(c3 != 0.0, 3, np.where(c2 != 0.0, 2, np.where(c1 != 0.0, 1, 0)))
    coef = np.stack([c0, c1, c2, c3], axis=1)
    for k in (1, 2, 3):
        sel = np.flatnonzero(deg == k)
        if len(sel) == 0:
            continue
        a = coef[sel, :k] / coef[sel, k:k + 1]          # monic: t^k + a_{k-1} t^{k-1} + ... + a_0
        comp = np.zeros((len(sel), k, k))
        comp[:, 0, :] = -a[:, ::-1]                      # numpy.roots' companion layout
        if k > 1:
            comp[:, np.arange(1, k), np.arange(k - 1)] = 1.0
        r = np.linalg.eigvals(comp)
        ok = (np.abs(r.imag) <= 1e-12 * np.maximum(1.0, np.abs(r.real))) & (r.real > 0.0)
        out[sel] = np.where(ok, r.real, np.inf).min(axis=1)
    return out.reshape(np.shape(c[0]))


def inversion_alpha(model, x, d):
    """Inversion filter: alpha = min(1, 0.9 min_e t_e), t_e = smallest positive root of
    det(Ds_e + t dDs_e) = 0.  Elements whose cubic provably has no root in
    (0, 1/0.9] are skipped before the (slow, per-element) root finding."""
    t = model.tets
    Ds = np.transpose(x[t][:, 1:] - x[t][:, :1], (0, 2, 1))
    dD = np.transpose(d[t][:, 1:] - d[t][:, :1], (0, 2, 1))
    c = det_poly(Ds, dD)
    T = 1.0 / FILTER_SAFETY
    # |c1| T + |c2| T^2 + |c3| T^3 < c0  =>  det > 0 on [0, T]: no root there
    cand = np.abs(c[1]) * T + np.abs(c[2]) * T ** 2 + np.abs(c[3]) * T ** 3 >= c[0]
    if not np.any(cand):
        return 1.0
    roots = smallest_positive_root([ci[cand] for ci in c])
    return float(min(1.0, FILTER_SAFETY * np.min(roots)))


def hlag_should_update(it, alphas, last_refresh, window=3, threshold=0.2, gap=5):
    """Refresh of the lagged elastic Hessian (§3.7.2; reading C4): always
    at the first Newton iteration of a timestep; afterwards when the moving average of the last
    `window` accepted step sizes drops below `threshold` and at least `gap` iterations passed since
    the last refresh."""
    if it == 0:
        return True
    if it - last_refresh < gap or not alphas:
        return False
    recent = alphas[-window:]
    return sum(recent) / len(recent) < threshold


@dataclasses.dataclass
class NewtonInfo:
    alpha: float
    alpha0: float
    ls_evals: int
    ds_norm: float
    converged: bool
    ls_failed: bool
    energy: float
    d: np.ndarray
    ds: np.ndarray
    df: np.ndarray
    cg_iters: int = 0


class OracleSim:
    """Timestep driver: begin_step / newton_iteration / end_step (Alg. 1)."""

    def __init__(self, scene, basis, n_cg=None, coarse_mode="exact", coarse_tol=1e-4, coarse_max_iter=None,
                 integrator="ie", cubature=None, lag=False, refine="jacobi", refine_tol=1e-2, refine_max_iter=100):
        self.coarse_mode, self.coarse_tol, self.coarse_max_iter = coarse_mode, coarse_tol, coarse_max_iter
        # NEXT-4: refinement PCG = fixed-count Jacobi (R5, default) or two-level to tolerance
        if refine == "two_level" and coarse_mode != "exact":
            raise ValueError("the two-level refinement needs the factorised coarse matrix (coarse_mode='exact')")
        self.refine, self.refine_tol, self.refine_max_iter = refine, refine_tol, refine_max_iter
        self.last_cg_iters = 0
        # NEXT-2 (§3.8, §3.7.2): cubature Hessian for the subspace solves, lagged Hessian for the
        # refinement (refresh policy: hlag_should_update)
        self.cubature, self.lag = cubature, lag
        self.lag_elastic = None
        self.lag_refreshes = 0
        self.step_iter, self.step_alphas, self.last_refresh = 0, [], 0
        self.integrator = integrator      # "ie" or "bdf2" (the first step is IE, no history)
        self.x_prev = self.v_prev = None
        self.scene = scene
        self.model = ip.make_model(scene)
        self.basis = basis
        self.Us = coarse.sms_matrix(self.model.X, basis)
        self.Ua = coarse.affine_matrix(self.model.X, basis)
        self.n_cg = basis.n_cg if n_cg is None else n_cg
        self.eps = scene.eps
        self.max_newton = scene.max_newton
        self.x = self.model.X.copy()
        self.v = np.zeros_like(self.x)
        self.elem_scale = None
        if cubature is not None:
            self.elem_scale = np.zeros(len(self.model.tets))
            self.elem_scale[cubature.elements] = cubature.weights / self.model.V[cubature.elements]

    def begin_step(self):
        self.step_iter, self.step_alphas, self.last_refresh = 0, [], 0
        self.x_t = self.x.copy()
        self.v_t = self.v.copy()
        if self.integrator == "bdf2" and self.x_prev is not None:
            self.model.alpha = 4.0 / 9.0
            self.xhat = ip.predictor_bdf2(self.model, self.x, self.v, self.x_prev, self.v_prev)
        else:
            self.model.alpha = 1.0
            self.xhat = ip.predictor(self.model, self.x, self.v)

    def direction(self, x):
        """(g, H, d_s, d_f, d) at x: Alg. 1 L229-238 -- full-space gradient, the subspace Hessian H
        (cubature-integrated with NEXT-2, else fully integrated: reading R3), H_lag for the
        refinement (lagged elastic part with NEXT-2, else H), d_s (Alg. 2), d_f = PCG(H_lag, -g - H d_s)."""
        m = self.model
        g = ip.gradient(m, x, self.xhat)
        H = ip.hessian(m, x, self.xhat, elem_scale=self.elem_scale).tocsr()
        if self.lag:
            if self.lag_elastic is None or hlag_should_update(self.step_iter, self.step_alphas, self.last_refresh):
                self.lag_elastic = ip.elastic_blocks(m, x)
                self.last_refresh = self.step_iter
                self.lag_refreshes += 1
            H_ref = ip.hessian(m, x, self.xhat, elastic=self.lag_elastic).tocsr()
        elif self.elem_scale is not None:
            H_ref = ip.hessian(m, x, self.xhat).tocsr()
        else:
            H_ref = H
        ds, da, Sa, S = subspace_direction(H, g, self.Ua, self.Us, self.coarse_mode, self.coarse_tol,
                                           self.coarse_max_iter)
        r = -g.ravel() - H @ ds
        if self.refine == "two_level":
            df, self.last_cg_iters = two_level_pcg(H_ref, r, self.Us, coarse.cholesky(S), self.refine_tol,
                                                   float(np.linalg.norm(g)), self.refine_max_iter)
        else:
            df, self.last_cg_iters = pcg(H_ref, r, self.n_cg), self.n_cg
        return g, H, ds, df, ds + df

    def newton_iteration(self):
        m = self.model
        x = self.x
        g, H, ds, df, d = self.direction(x)
        d3 = d.reshape(-1, 3)
        a0 = min(ccd_alpha(m, x, d3), inversion_alpha(m, x, d3))
        alpha = a0
        evals = 0
        failed = False
        while True:
            evals += 1
            if ip.energy_difference(m, x, d3, alpha, self.xhat) < 0.0:
                break
            alpha *= LS_SHRINK
            if alpha < LS_MIN:
                failed = True
                break
        if not failed:
            self.x = x + alpha * d3
        self.step_alphas.append(alpha if not failed else 0.0)
        self.step_iter += 1
        ds_norm = float(np.linalg.norm(ds))
        conv = ds_norm / (m.h * m.n) < self.eps
        return NewtonInfo(alpha, a0, evals, ds_norm, conv, failed,
                          ip.energy(m, self.x, self.xhat), d, ds, df, self.last_cg_iters)

    def end_step(self):
        h = self.model.h
        if self.model.alpha != 1.0:
            # BDF2 (reading C2): a = 9/(4h^2)(x - xtilde) with xtilde the predictor without
            # the folded gravity, v = (4v^t - v^{t-1})/3 + (2h/3) a
            xtilde = self.xhat - (4.0 / 9.0) * h ** 2 * self.model.gravity[None, :]
            a = 9.0 / (4.0 * h ** 2) * (self.x - xtilde)
            v_new = (4.0 * self.v_t - self.v_prev) / 3.0 + (2.0 * h / 3.0) * a
        else:
            v_new = (self.x - self.x_t) / h
        self.x_prev, self.v_prev = self.x_t, self.v_t
        self.v = v_new

    def timestep(self):
        self.begin_step()
        infos = []
        for _ in range(self.max_newton):
            info = self.newton_iteration()
            infos.append(info)
            if info.converged or info.ls_failed:
                break
        self.end_step()
        return infos
