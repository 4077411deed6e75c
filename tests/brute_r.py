"""Brute-force, high-precision transcription of the reading R -- TEST INFRASTRUCTURE ONLY.

SURVEY.md 8(c.3), row "Implementation of R": one or two CSPH-TVD steps on tiny grids,
evaluated in 50-digit mpmath arithmetic straight from the text of DESIGN.md section 3
(which restates PAPER.md:224-238, K1..K8, and Eqs. 1-7), to be compared with the fp64
oracle (oracle/csph_oracle.c).  It shares nothing with the oracle: no import, no
table, no helper.  It is also built differently, so that a slip copied from one to the
other is unlikely:

* cell-centred and lazy -- every quantity of R is a memoised function of a cell or a
  face index (``Hh(i, j)``, ``flux_x(i, j)``), evaluated on demand, never a loop nest
  over an array;
* ghosts are index reflections (``_src``) applied on every read, never copies;
* x^(-1/3) is the exact real cube root (the oracle's pinned recipe is within 2 ulp);
* every branch decision of R goes through ``_decide``, which records how far the
  deciding value is from its threshold, so that a caller can reject random inputs that
  sit within rounding of a threshold ("inputs chosen away from every
  branch threshold"); at such inputs a correct fp64 implementation may legitimately
  take the other branch.

Time levels, as DESIGN.md 3.3-3.6 fixes them:
  K1 (w, eta, r, u, v) and K2 (Phi^n, gamma) from state n; K4 the predictor to
  t_{n+1/2} (H_half, u~, v~); K5 forces from eta_half = H_half + b with the step-n mask;
  K6 Q^L; K7 reconstructs the n-level eta and H and the half-step u~, v~, and the
  sediment gate / film cut-off use the n-level H; K8 the update; step 9 the maxima of
  the new state for Eq.7.
"""
from __future__ import annotations

from functools import lru_cache

import mpmath as mp

DPS = 50


def _m(x) -> mp.mpf:
    """Exact conversion of a float (or int) to a 50-digit mpf."""
    return mp.mpf(x)


class Margins:
    """Smallest relative distance of a decided value from its threshold.  Exact ties
    (distance 0) are structural (e.g. a dry cell's H* = max(0, 0)) and both sides meet
    them exactly, so they are counted apart."""

    def __init__(self):
        self.min_rel = mp.inf
        self.where = None
        self.ties = 0

    def note(self, diff, scale, tag):
        if diff == 0:
            self.ties += 1
            return
        s = abs(scale)
        r = abs(diff) / s if s > 0 else mp.inf
        if r < self.min_rel:
            self.min_rel = r
            self.where = tag


class BruteR:
    """One domain of nx x ny cells with solid walls (1) or open edges (2) per side
    (xlo, xhi, ylo, yhi), parameters as in oracle.Params (a plain dict here)."""

    def __init__(self, nx, ny, h, prm: dict, H, Qx, Qy, b, psi=None, bc=(1, 1, 1, 1),
                 n_field=None, beta=None, src=None):
        mp.mp.dps = DPS
        self.nx, self.ny = nx, ny
        self.h = _m(h)
        self.p = {k: (v if isinstance(v, int) and not isinstance(v, bool) else _m(v))
                  for k, v in prm.items()}
        self.bc = bc
        self.mg = Margins()

        def grid(a, default=0.0):
            return {(i, j): _m(a[j][i] if a is not None else default)
                    for j in range(ny) for i in range(nx)}

        self.H, self.Qx, self.Qy, self.b = grid(H), grid(Qx), grid(Qy), grid(b)
        # Eq.1: W = 1/(1 - psi), once per cell
        ps = grid(psi) if psi is not None else {k: _m(0) for k in self.H}
        self.W = {k: 1 / (1 - v) for k, v in ps.items()}
        nm = self.p["n_manning"]
        self.nM = grid(n_field) if n_field is not None else {k: nm for k in self.H}
        self.fric = n_field is not None or nm > 0
        self.beta = grid(beta) if beta is not None else None
        self.srcf = grid(src) if src is not None else None
        if self.beta is None and self.srcf is not None:
            self.beta = {k: _m(0) for k in self.H}
        if self.srcf is None and self.beta is not None:
            self.srcf = {k: _m(0) for k in self.H}
        self.t = _m(0)
        self.taus, self.lims = [], []

    # ---------------------------------------------------------------- ghosts
    def _src(self, i, j):
        """Reflection of a (possibly ghost) index onto the owned cell it copies, and the
        signs of the x and y momenta there (wall = mirror with the
        normal momentum negated; open = the boundary cell unchanged)."""
        sx = sy = 1
        if i < 0:
            if self.bc[0] == 1:
                i, sx = -1 - i, -1
            else:
                i = 0
        elif i >= self.nx:
            if self.bc[1] == 1:
                i, sx = 2 * self.nx - 1 - i, -1
            else:
                i = self.nx - 1
        if j < 0:
            if self.bc[2] == 1:
                j, sy = -1 - j, -1
            else:
                j = 0
        elif j >= self.ny:
            if self.bc[3] == 1:
                j, sy = 2 * self.ny - 1 - j, -1
            else:
                j = self.ny - 1
        return i, j, sx, sy

    def _cell(self, S, i, j):
        """(H, Qx, Qy, b, W, n_M) of any index of the state S = (H, Qx, Qy, b)."""
        a, c, sx, sy = self._src(i, j)
        k = (a, c)
        return S[0][k], sx * S[1][k], sy * S[2][k], S[3][k], self.W[k], self.nM[k]

    # ------------------------------------------------------------ decisions
    def _decide(self, x, y, scale, tag):
        """x > y, recording the margin |x - y| / scale."""
        self.mg.note(x - y, scale, tag)
        return x > y

    def _pos(self, x, scale, tag):
        """max(0, x): the kink at 0 is a decision (the dry side of a hydrostatic face)."""
        self.mg.note(x, scale, tag)
        return x if x > 0 else _m(0)

    # ------------------------------------------------------------ closures
    def _grass_pow(self, s2):
        """|v|^m of Eq.3, exact (the real exponent m_real when it is >= 0)."""
        if self.p.get("m_real", -1) >= 0:
            return mp.power(s2, self.p["m_real"] / 2) if s2 > 0 else (
                _m(1) if self.p["m_real"] == 0 else _m(0))
        m = self.p["m_grass"]
        return mp.power(mp.sqrt(s2), m) if m % 2 else mp.power(s2, m // 2)

    def _A(self, H, nM):
        """A_J: the constant, or Eq.4 at the local depth H (0 on a dry cell)."""
        p = self.p
        if p["aj_mode"] == 0:
            return p["A_J"]
        if not self._decide(H, p["eps_dry"], p["eps_dry"], "Eq4 wet"):
            return _m(0)
        return (mp.mpf("0.05") * nM ** 3) / ((p["s_rel"] - 1) * mp.sqrt(p["g"] * H) * p["d50"])

    def _mobile(self, s2, H, tag):
        """Eq.5 gate (reading #6: |v| > v_k <=> s2^3 > kappa H) and the film cut-off of
        reading #31 (H > h_bed_min; h_bed_min < 0 means d50)."""
        p = self.p
        kappa = p["C_Sh"] ** 6 * p["d50"] ** 2
        ok = True
        if p["C_Sh"] != 0:
            ok = self._decide(s2 ** 3, kappa * H, kappa * H + s2 ** 3, "gate " + tag)
        hb = p["h_bed_min"] if p["h_bed_min"] >= 0 else p["d50"]
        film = self._decide(H, hb, hb if hb > 0 else _m(1), "film " + tag)
        return ok and film

    # ------------------------------------------------------------ one step
    def maxima(self, S):
        """Step 9 / initial reduction: maxima over owned wet cells."""
        p = self.p
        M1 = M2 = M3 = _m(0)
        for j in range(self.ny):
            for i in range(self.nx):
                H, Qx, Qy, _, W, nM = self._cell(S, i, j)
                if not self._decide(H, p["eps_dry"], p["eps_dry"], "M wet"):
                    continue
                u, v = Qx / H, Qy / H
                s2 = u * u + v * v
                M1 = max(M1, s2)
                M2 = max(M2, mp.sqrt(s2) + mp.sqrt(p["g"] * H))
                if self._mobile(s2, H, "M"):
                    M3 = max(M3, self._A(H, nM) * self._grass_pow(s2) * mp.sqrt(s2) * W)
        return M1, M2, M3

    def tau_of(self, M):
        """Eq.7, reading #9: tau = K min(h/(2 sqrt M1), h/M2, h^2/(2 M3))."""
        p, h = self.p, self.h
        terms = [h / (2 * mp.sqrt(M[0])) if M[0] > 0 else mp.inf,
                 h / M[1] if M[1] > 0 else mp.inf,
                 h * h / (2 * M[2]) if M[2] > 0 else mp.inf]
        lim = min(range(3), key=lambda k: (terms[k], k))
        tau = p["K"] * terms[lim]
        if p["dt_max"] < tau:
            tau, lim = p["dt_max"], 3
        if not mp.isfinite(tau):
            raise ValueError("all dry (EDRY)")
        for k in range(3):  # the limiter choice: ties are decisions too
            if k != lim and mp.isfinite(terms[k]) and lim < 3:
                self.mg.note(terms[k] - terms[lim], terms[lim], "Eq7 limiter")
        return tau, lim

    def step(self):
        S = (self.H, self.Qx, self.Qy, self.b)
        tau, lim = self.tau_of(self.maxima(S))
        new = self._advance(S, tau)
        self.H, self.Qx, self.Qy, self.b = new
        self.t += tau
        self.taus.append(tau)
        self.lims.append(lim)
        return tau, lim

    def probe(self, i, j):
        """(H_n, H_half, u~, v~) of cell (i, j) in the coming step (no state change)."""
        S = (self.H, self.Qx, self.Qy, self.b)
        tau, _ = self.tau_of(self.maxima(S))
        return self._advance(S, tau, probe=(i, j))

    def _advance(self, S, tau, probe=None):
        p = self.p
        g, eps, h = p["g"], p["eps_dry"], self.h
        theta = tau / 2
        lam = tau / h
        half = mp.mpf("0.5")
        cell = lru_cache(maxsize=None)(lambda i, j: self._cell(S, i, j))

        # ---- K1: mask, eta, r, u, v at t_n
        @lru_cache(maxsize=None)
        def k1(i, j):
            H, Qx, Qy, b, _, _ = cell(i, j)
            w = self._decide(H, eps, eps, "K1 wet")
            if not w:
                return False, H + b, _m(0), _m(0), _m(0)
            r = 1 / H
            return True, H + b, r, Qx * r, Qy * r

        def face_P(etaL, bL, etaR, bR, tag):
            """K2/K5 face pressure term, hydrostatic form (DESIGN.md 3.3 step 2)."""
            bs = max(bL, bR)
            sc = abs(etaL) + abs(etaR) + abs(bs)
            HL = self._pos(etaL - bs, sc, tag)
            HR = self._pos(etaR - bs, sc, tag)
            return (g / (2 * h)) * half * (HL + HR) * (HR - HL)

        # ---- K2: forces at t_n and Manning gamma (reading #19)
        @lru_cache(maxsize=None)
        def k2(i, j):
            w, eta, r, u, v = k1(i, j)
            if not w:
                return _m(0), _m(0), _m(0)
            b = cell(i, j)[3]

            def nb(a, c):
                return k1(a, c)[1], cell(a, c)[3]

            eE, bE = nb(i + 1, j); eW, bW = nb(i - 1, j)
            eN, bN = nb(i, j + 1); eS, bS = nb(i, j - 1)
            PE = face_P(eta, b, eE, bE, "K2"); PW = face_P(eW, bW, eta, b, "K2")
            PN = face_P(eta, b, eN, bN, "K2"); PS = face_P(eS, bS, eta, b, "K2")
            gam = _m(0)
            if self.fric:
                H, nM = cell(i, j)[0], cell(i, j)[5]
                gam = g * nM * nM * mp.sqrt(u * u + v * v) / (H * mp.cbrt(H))
            return -(PE + PW), -(PN + PS), gam

        # ---- K4: predictor to t_{n+1/2}
        @lru_cache(maxsize=None)
        def k4(i, j):
            w, _, r, _, _ = k1(i, j)
            H, Qx, Qy = cell(i, j)[:3]
            if not w:
                return H, _m(0), _m(0)  # a dry cell keeps H and holds no velocity
            div = ((k1(i + 1, j)[3] - k1(i - 1, j)[3]) + (k1(i, j + 1)[4] - k1(i, j - 1)[4])) / (2 * h)
            phx, phy, gam = k2(i, j)
            f = 1 / (1 + theta * gam)
            return H * (1 - theta * div), (Qx + theta * phx) * f * r, (Qy + theta * phy) * f * r

        # ---- K5: forces at t_{n+1/2} on eta_half, step-n mask
        @lru_cache(maxsize=None)
        def k5(i, j):
            if not k1(i, j)[0]:
                return _m(0), _m(0)

            def eh(a, c):
                return k4(a, c)[0] + cell(a, c)[3], cell(a, c)[3]

            ec, bc = eh(i, j)
            eE, bE = eh(i + 1, j); eW, bW = eh(i - 1, j)
            eN, bN = eh(i, j + 1); eS, bS = eh(i, j - 1)
            return (-(face_P(ec, bc, eE, bE, "K5") + face_P(eW, bW, ec, bc, "K5")),
                    -(face_P(ec, bc, eN, bN, "K5") + face_P(eS, bS, ec, bc, "K5")))

        if probe is not None:
            return (cell(*probe)[0],) + k4(*probe)

        # ---- K6: corrector momenta
        def k6(i, j):
            if not k1(i, j)[0]:
                return _m(0), _m(0)
            Qx, Qy = cell(i, j)[1:3]
            f = 1 / (1 + tau * k2(i, j)[2])
            px, py = k5(i, j)
            return (Qx + tau * px) * f, (Qy + tau * py) * f

        # ---- per-cell gated Grass flux (Eqs. 3, 5; n-level H) on u~, v~
        @lru_cache(maxsize=None)
        def j0(i, j):
            _, ut, vt = k4(i, j)
            H, nM = cell(i, j)[0], cell(i, j)[5]
            s2 = ut * ut + vt * vt
            if not self._mobile(s2, H, "K7"):
                return _m(0), _m(0), _m(0)
            a = self._A(H, nM) * self._grass_pow(s2)
            return a * ut, a * vt, a * mp.sqrt(s2)

        def minmod(a, b):
            if a > 0 and b > 0:
                return min(a, b)
            if a < 0 and b < 0:
                return max(a, b)
            return _m(0)

        # ---- K7: one face between L and R along an axis
        @lru_cache(maxsize=None)
        def flux(axis, i, j):
            """Face between cell (i,j) - e_axis (side L, '-') and (i,j) (side R, '+').
            Returns (F_mass, F_normal momentum, F_tangential momentum, J_bed)."""
            di, dj = (1, 0) if axis == 0 else (0, 1)
            cs = [(i + k * di, j + k * dj) for k in (-2, -1, 0, 1)]  # LL, L, R, RR

            def q(c):
                _, eta, _, _, _ = k1(*c)
                H = cell(*c)[0]
                _, ut, vt = k4(*c)
                un, uq = (ut, vt) if axis == 0 else (vt, ut)
                return [eta, H, un, uq]

            LL, L, R, RR = (q(c) for c in cs)
            wL, wR = k1(*cs[1])[0], k1(*cs[2])[0]
            if not wL and not wR:
                return _m(0), _m(0), _m(0), _m(0)
            qm = [L[k] + half * minmod(L[k] - LL[k], R[k] - L[k]) for k in range(4)]
            qp = [R[k] - half * minmod(R[k] - L[k], RR[k] - R[k]) for k in range(4)]
            # hydrostatic step
            bm, bp = qm[0] - qm[1], qp[0] - qp[1]
            bs = max(bm, bp)
            sc = abs(qm[0]) + abs(qp[0]) + abs(bs)
            Hm = self._pos(qm[0] - bs, sc, "K7 H*-")
            Hp = self._pos(qp[0] - bs, sc, "K7 H*+")
            F = [_m(0)] * 3
            if Hm > 0 or Hp > 0:
                um, utm, up, utp = qm[2], qm[3], qp[2], qp[3]
                FL = [Hm * um, Hm * um * um, Hm * um * utm]
                FR = [Hp * up, Hp * up * up, Hp * up * utp]
                UL = [Hm, Hm * um, Hm * utm]
                UR = [Hp, Hp * up, Hp * utp]
                cm, cp = mp.sqrt(g * Hm), mp.sqrt(g * Hp)
                if Hm > 0 and Hp > 0:
                    SL, SR = min(um - cm, up - cp), max(um + cm, up + cp)
                elif Hm > 0:  # + side dry: a rarefaction into the dry bed
                    SL, SR = um - cm, um + 2 * cm
                else:
                    SL, SR = up - 2 * cp, up + cp
                if SL >= 0:
                    F = FL
                elif SR <= 0:
                    F = FR
                else:
                    F = [(SR * FL[k] - SL * FR[k] + SL * SR * (UR[k] - UL[k])) / (SR - SL)
                         for k in range(3)]
            # sediment face flux, Eq.2 vector reading #4 with the donor cell
            JL, JR = j0(*cs[1]), j0(*cs[2])
            ax = 0 if axis == 0 else 1
            unL, unR = L[2], R[2]
            us = unL + unR
            self.mg.note(us, abs(unL) + abs(unR), "donor")
            if us > 0:
                Jn, Ja = JL[ax], JL[2]
            elif us < 0:
                Jn, Ja = JR[ax], JR[2]
            else:
                Jn, Ja = (JL[ax] + JR[ax]) / 2, (JL[2] + JR[2]) / 2
            bL, bR = cell(*cs[1])[3], cell(*cs[2])[3]
            Jf = Jn - p["C_J"] * Ja * (bR - bL) / h
            return F[0], F[1], F[2], Jf

        # ---- K8 (Eqs. 1, 6): conservative update of the owned cells
        Hn, Qxn, Qyn, bn = {}, {}, {}, {}
        src_q = p["q_plus"] - p["q_minus"]
        for j in range(self.ny):
            for i in range(self.nx):
                H, _, _, b, W, _ = cell(i, j)
                fE, fW = flux(0, i + 1, j), flux(0, i, j)
                gN, gS = flux(1, i, j + 1), flux(1, i, j)
                d = [(fE[k] - fW[k]) for k in range(4)]
                e = [(gN[k] - gS[k]) for k in range(4)]
                # x-faces carry (mass, Qx, Qy); y-faces carry (mass, Qy, Qx): normal first
                dH = d[0] + e[0]
                dQx = d[1] + e[2]
                dQy = d[2] + e[1]
                dJ = d[3] + e[3]
                QLx, QLy = k6(i, j)
                H2 = H - lam * dH
                Qx2 = QLx - lam * dQx
                Qy2 = QLy - lam * dQy
                if self.beta is not None:
                    a = 1 / (1 + tau * self.beta[(i, j)])
                    H2 = (H2 + tau * self.srcf[(i, j)]) * a
                    Qx2, Qy2 = Qx2 * a, Qy2 * a
                b2 = b - lam * W * dJ + tau * W * src_q
                if not self._decide(H2, eps, eps, "K8 wet"):
                    Qx2 = Qy2 = _m(0)
                Hn[(i, j)], Qxn[(i, j)], Qyn[(i, j)], bn[(i, j)] = H2, Qx2, Qy2, b2
        return Hn, Qxn, Qyn, bn

    # ---------------------------------------------------------------- output
    def state(self):
        """(H, Qx, Qy, b) as nested lists of mpf, [j][i]."""
        return [[[F[(i, j)] for i in range(self.nx)] for j in range(self.ny)]
                for F in (self.H, self.Qx, self.Qy, self.b)]
