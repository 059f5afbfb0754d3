"""CPU restatement of the reference's fast solver (interpolation space-time FMM).

TEST INFRASTRUCTURE ONLY (imported by tests/ and bench.py's baseline legs).

The reference `fast_march` (pkg/src/tdwavebem/fmm.py:422-544) crashes as
shipped and is inaccurate.  This module restates its time loop
with the seven corrections of SURVEY.md 8(c):
  1. P2M contraction tau[elems] @ p2m_tau (fmm.py:517-518),
  2. node-offset sign of the kernel samples (fmm.py:87)        -> fmm_plan.kernel_tensor,
  3. source interval k_src = floor((t_src + dt) / I)            (fmm.py:512),
  4. source temporal weights with extrapolate = 2 dt / I        (fmm.py:514),
  5. extra-list break test on floor((t_src + dt) / I_L)          (fmm.py:464),
  6. extra-list lag count floor(I_L / dt) + 2                    (fmm.py:226),
  7. marginal margin c I_L, reach c (I_L + dt) + 2 rho           (fmm_tree.py:202, 206).
The structure follows fmm.py: _do_m2l (:329-368, near-future lags + derivative
operators + the Algorithm-1 recurrence), _tick (:371-419, M2M up while the
time-half bit is 1, L2L down into inherit slots), run (:422-531).  The near
field is the reference's lag CSR restricted to near pairs with window gamma_near
(marching.py:132-181 / fmm.py:213-235), built from the C oracle's coefficient
table; the lag-1 system is solved with scipy's SuperLU as in the reference.

The operator data (tree, interpolation rows, Toeplitz tensors) comes from
paper_2111_05205_b200.fmm_plan, whose pieces are pinned against the reference
by tests/test_fmm_host.py (bit-exact tree, golden interpolation/kernel data).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import oracle

W_D = {1: [1.0, -2.0, 1.0], 2: [0.5, -1.5, 1.5, -0.5],
       3: [1.0 / 6, -2.0 / 3, 1.0, -2.0 / 3, 1.0 / 6]}


def _arrival(cent, radii, ci, cj, c, dt):
    dist = np.linalg.norm(cent[ci] - cent[cj], axis=1)
    dist = np.maximum(dist - radii[cj], 0.0)
    return np.maximum(np.ceil(dist / (c * dt)).astype(np.int32) - 1, 1)


def lag_csr(spec, ii, jj, G):
    """Per-lag CSR (U[g-1], W[g-1]), g = 1..G, of the pairs (ii, jj): every pair
    already arrived by lag g (marching.py:93-181)."""
    mesh = spec.mesh
    ns = mesh.n_elements
    c, dt, d = spec.c, spec.basis.dt, spec.basis.d
    cent = mesh.centroids
    radii = mesh.element_radii()
    v0, v1, v2 = mesh.element_vertices()
    arr = _arrival(cent, radii, ii, jj, c, dt)
    keep = arr <= G
    ii, jj, arr = ii[keep], jj[keep], arr[keep]
    order = np.argsort(arr, kind="stable")
    ii, jj, arr = ii[order], jj[order], arr[order]
    U, W = [], []
    for g in range(1, G + 1):
        live = int(np.searchsorted(arr, g, side="right"))
        bi, bj = ii[:live], jj[:live]
        s = np.full(live, g * c * dt)
        if live:
            if spec.bie == "obie":
                u, w = oracle.coeff_table(cent[bi], v0[bj], v1[bj], v2[bj], mesh.normals[bj], s, d, c, dt)
            else:
                u, w = oracle.coeff_table(cent[bi], v0[bj], v1[bj], v2[bj], mesh.normals[bj], s, d,
                                          c, dt, "bm", -mesh.normals[bi])
        else:
            u = w = np.zeros(0)
        U.append(sp.csr_matrix((u, (bi, bj)), shape=(ns, ns)))
        W.append(sp.csr_matrix((w, (bi, bj)), shape=(ns, ns)))
    return U, W


class FmmOracle:
    def __init__(self, spec, plan):
        self.spec, self.plan = spec, plan
        self.d = spec.basis.d
        self.w = np.array(W_D[self.d])
        self.near_U, self.near_W = lag_csr(spec, plan.near_i, plan.near_j, plan.gamma_near)
        self.extra = {L: lag_csr(spec, ei, ej, lags) + (lags,) for L, (ei, ej, lags) in plan.extra.items()}
        w0 = self.w[0]
        phi = spec.phi
        A = self.near_W[0].multiply(phi[None, :]) - self.near_U[0].multiply((1.0 - phi)[None, :])
        self.A = (w0 * A).tocsc()
        self.lu = spla.splu(self.A)
        ps, pt, mu = plan.ps, plan.pt, plan.mu
        self.nd = ps ** 3 * pt
        self.state = {}
        for L, ops in plan.levels.items():
            n = ops.n_cells
            self.state[L] = dict(own=np.zeros((mu + 3, n, self.nd)), inherit=np.zeros((4, n, self.nd)),
                                 deriv=np.zeros((self.d, n, self.nd)),
                                 aux={(p, m): np.zeros((n, self.nd)) for p in range(2, self.d + 1)
                                      for m in range(p - 1)},
                                 acc=np.zeros((n, self.nd)))
        # dense operators per (level, offset): op 0..mu = lags 1..mu+1, mu+1.. = p=1..d,
        # stacked (nops, nd, nd); the interaction pairs of a level grouped by offset
        # (an observer appears at most once per offset, so a group's updates never collide)
        from paper_2111_05205_b200.fmm_plan import dense_operator
        self.ops = {}
        self.groups = {}
        for L, ops in plan.levels.items():
            mats = []
            for o in range(len(ops.offsets)):
                K0 = ops.K0[o].reshape(2 * ps - 1, 2 * ps - 1, 2 * ps - 1, -1)
                row = [dense_operator(K0, ps, pt, l * (pt - 1)) for l in range(1, mu + 2)]
                for p in range(1, self.d + 1):
                    Kp = ops.Kp[p - 1][o].reshape(2 * ps - 1, 2 * ps - 1, 2 * ps - 1, -1)
                    row.append(dense_operator(Kp, ps, pt, pt - 1))
                # (nd, nops * nd): Y = Ms @ stack gives every operator's result side by side
                mats.append(np.ascontiguousarray(np.concatenate(row, axis=0).T))
            self.ops[L] = mats
            obs = np.repeat(np.arange(ops.n_cells), np.diff(ops.obs_ptr))
            src, off = np.asarray(ops.il_src), np.asarray(ops.il_off)
            order = np.argsort(off, kind="stable")
            bounds = np.searchsorted(off[order], np.arange(len(ops.offsets) + 1))
            self.groups[L] = [(obs[order[bounds[o]:bounds[o + 1]]], src[order[bounds[o]:bounds[o + 1]]])
                              for o in range(len(ops.offsets))]

    # -- translation operators (fmm.py:314-326): index order (a1, a2, a3, m), applied
    #    to all cells of one octant at once
    def _transfer_moment(self, M, octant, half):
        P = self.plan
        X = M.reshape(-1, P.ps, P.ps, P.ps, P.pt)
        X = np.einsum("pa,nabcm->npbcm", P.t_space[octant[0]], X)
        X = np.einsum("qb,npbcm->npqcm", P.t_space[octant[1]], X)
        X = np.einsum("rc,npqcm->npqrm", P.t_space[octant[2]], X)
        X = np.einsum("sm,npqrm->npqrs", P.t_time[half], X)
        return X.reshape(len(X), -1)

    def _transfer_local(self, Lp, octant, half):
        P = self.plan
        X = Lp.reshape(-1, P.ps, P.ps, P.ps, P.pt)
        X = np.einsum("pa,npbcm->nabcm", P.t_space[octant[0]], X)
        X = np.einsum("qb,naqcm->nabcm", P.t_space[octant[1]], X)
        X = np.einsum("rc,nabrm->nabcm", P.t_space[octant[2]], X)
        X = np.einsum("sm,nabcs->nabcm", P.t_time[half], X)
        return X.reshape(len(X), -1)

    def _octant_groups(self, ops):
        oc = np.asarray(ops.octant)
        key = oc[:, 0] + 2 * oc[:, 1] + 4 * oc[:, 2]
        return [(np.nonzero(key == g)[0], oc[np.nonzero(key == g)[0][0]]) for g in range(8) if (key == g).any()]

    def _do_m2l(self, L, k, moments):
        """Near-future lags, derivative operators and the Algorithm-1 recurrence
        (fmm.py:329-368), one dense contraction per offset group."""
        P, st, ops = self.plan, self.state[L], self.plan.levels[L]
        mu, d, nd = P.mu, self.d, self.nd
        T = P.c * ops.interval
        ring = mu + 3
        tmp = np.zeros((d, ops.n_cells, nd))
        for oi, (obs, src) in enumerate(self.groups[L]):
            if len(obs) == 0:
                continue
            Y = moments[src] @ self.ops[L][oi]                   # (n, nops * nd), BLAS
            for l in range(1, mu + 2):
                if ops.dark[oi, l - 1]:
                    continue
                st["own"][(k + l) % ring][obs] += Y[:, (l - 1) * nd:l * nd]
            for p in range(1, d + 1):
                tmp[p - 1][obs] += Y[:, (mu + p) * nd:(mu + p + 1) * nd]
        from paper_2111_05205_b200.fmm_plan import cmp_coeff
        for p in range(1, d + 1):
            upd = tmp[p - 1].copy()
            for m in range(p - 1):
                upd = upd + cmp_coeff(p, m, k) * st["aux"][(p, m)]
            st["deriv"][p - 1] += upd
        new = st["own"][(k + mu + 1) % ring].copy()
        for p in range(1, d + 1):
            new += st["deriv"][p - 1] * T ** p
        st["own"][(k + mu + 2) % ring] = new
        for p in range(2, d + 1):
            for m in range(p - 1):
                st["aux"][(p, m)] += tmp[p - 1] * float(k) ** m

    def _tick(self, k_leaf):
        """Close leaf interval k_leaf (fmm.py:371-419): M2L at the leaf, M2M up while
        the time-half bit is 1 (M2L at each closed level), L2L down into the
        children's inherit slots."""
        P = self.plan
        leaf = P.leaf
        completed = [leaf]
        moments = self.state[leaf]["acc"].copy()
        self.state[leaf]["acc"][:] = 0.0
        self._do_m2l(leaf, k_leaf, moments)
        cur_k, L = k_leaf, leaf
        while L - 1 >= 2:
            ops = P.levels[L]
            pst = self.state[L - 1]
            half = cur_k & 1
            for cells, oc in self._octant_groups(ops):
                np.add.at(pst["acc"], np.asarray(ops.parent)[cells],
                          self._transfer_moment(moments[cells], oc, half))
            if half == 0:
                break
            cur_k >>= 1
            L -= 1
            completed.append(L)
            moments = self.state[L]["acc"].copy()
            self.state[L]["acc"][:] = 0.0
            self._do_m2l(L, cur_k, moments)
        for L in sorted(completed):
            if L + 1 > leaf:
                continue
            k_level = k_leaf >> (leaf - L)
            st = self.state[L]
            ring = P.mu + 3
            total = st["own"][(k_level + 1) % ring] + st["inherit"][(k_level + 1) % 4]
            child = P.levels[L + 1]
            cst = self.state[L + 1]
            par = np.asarray(child.parent)
            for cells, oc in self._octant_groups(child):
                for half in (0, 1):
                    kc = 2 * (k_level + 1) + half
                    cst["inherit"][kc % 4, cells] = self._transfer_local(total[par[cells]], oc, half)

    def run(self, u_known, q_known, threshold=1e6):
        spec, P = self.spec, self.plan
        from paper_2111_05205_b200.fmm_plan import step_schedule
        nt, ns, d = spec.nt, spec.mesh.n_elements, self.d
        sched = step_schedule(P, nt)
        w = self.w
        phi = spec.phi
        u = np.zeros((nt - 1, ns))
        q = np.zeros((nt - 1, ns))
        tau = np.zeros((nt - 1, ns))
        sig = np.zeros((nt - 1, ns))
        n_lags = P.gamma_near
        last_tick = -1
        leaf = P.leaf
        ring = P.mu + 3
        status, n_steps = "stable", 0
        rhs = []

        def stock(arr, beta, kmax):
            acc = np.zeros(ns)
            for k in range(kmax + 1):
                acc += w[k] * arr[beta - k]
            return acc

        for alpha in range(1, nt):
            beta0 = alpha - 1
            while last_tick < sched["ticks_before"][alpha]:
                self._tick(last_tick + 1)
                last_tick += 1
            beta_star = alpha - n_lags
            uk, qk = u_known[beta0], q_known[beta0]
            tau_t = w[0] * qk * phi
            sig_t = w[0] * uk * (1.0 - phi)
            for k in range(1, min(d + 1, beta0) + 1):
                tau_t += w[k] * q[beta0 - k]
                sig_t += w[k] * u[beta0 - k]
            b = self.near_U[0] @ tau_t - self.near_W[0] @ sig_t
            for g in range(2, min(alpha, n_lags) + 1):
                beta = alpha - g
                if beta - beta_star <= d:
                    kmax = min(d + 1, beta - beta_star, beta)
                    tb, sb = stock(q, beta, kmax), stock(u, beta, kmax)
                else:
                    tb, sb = tau[beta], sig[beta]
                b += self.near_U[g - 1] @ tb - self.near_W[g - 1] @ sb
            for L, (Ue, We, lags) in self.extra.items():
                for g in range(1, sched["extra_gmax"][L][alpha] + 1):
                    tb, sb = (tau_t, sig_t) if g == 1 else (tau[alpha - g], sig[alpha - g])
                    b += Ue[g - 1] @ tb - We[g - 1] @ sb
            # far field through the leaf locals (L2P)
            ko = sched["k_obs"][alpha]
            st = self.state[leaf]
            Lt = st["own"][ko % ring] + st["inherit"][ko % 4]          # (ncell, nd)
            flat = Lt.reshape(len(Lt), -1, P.pt)
            cell = P.elem_cell
            if spec.bie == "obie":
                b += np.einsum("ea,eam,m->e", P.l2p_val, flat[cell], sched["wt"][alpha])
            else:
                b += np.einsum("ea,eam,m->e", P.l2p_bm, flat[cell], sched["wt"][alpha])
                b -= np.einsum("ea,eam,m->e", P.l2p_val, flat[cell], sched["dwt"][alpha])
            rhs.append(b.copy())
            x = self.lu.solve(b)
            if np.linalg.norm(self.A @ x - b) > 1e-10 * max(np.linalg.norm(b), 1e-300):
                raise RuntimeError(f"step {alpha}: residual")
            u[beta0] = np.where(phi == 1.0, x, uk)
            q[beta0] = np.where(phi == 1.0, qk, x)
            kk = min(d + 1, beta0)
            tau[beta0], sig[beta0] = stock(q, beta0, kk), stock(u, beta0, kk)
            n_steps = alpha
            # P2M of this step's source into the leaf moment of interval k_src
            spat = P.p2m_tau * tau[beta0][:, None] - P.p2m_sig * sig[beta0][:, None]   # (ns, ps^3)
            cm = np.zeros((len(st["acc"]), P.ps ** 3))
            np.add.at(cm, cell, spat)
            st["acc"] += np.einsum("cs,t->cst", cm, sched["wts"][alpha]).reshape(len(cm), -1)
            if np.max(np.abs(x)) > threshold:
                status = "unstable"
                break
        return dict(u=u, q=q, tau=tau, sigma=sig, n_steps=n_steps, status=status, rhs=np.array(rhs))
