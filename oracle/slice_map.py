"""Per-pixel maps of a time slice -- TEST INFRASTRUCTURE ONLY.

Plain fp64 restatement of what a time slice of the stream does to one pixel's
Alg. 2 state, written out event by event:

  no event in the slice   : (S, T) unchanged;
  events e_1 .. e_n       : S1 = clamp((S + p_1 C) d(t_1 - T))
                            S' = g_n( ... g_2(S1) ... ),  T' = t_n
  g_k(s) = clamp(d_k s + d_k p_k C, S_min, S_max),  d_k = d(t_k - t_{k-1})  (Eq. 4 at P:160, Eq. 13 at P:218);
  decay-first variant (reading A20): S1 = clamp(S d(t_1 - T) + p_1 C), g_k(s) = clamp(d_k s + p_k C).

The later events compose into one clamped affine map G(s) = min(max(a s + c, lo), hi)
with the monoid product of SURVEY section 0,
  F o G = (aF aG, aF cG + cF, clamp(aF loG + cF, loF, hiF), clamp(aF hiG + cF, loF, hiF)),
so a slice is summarised per pixel by (n, t_first, p_first, G, t_last); two
consecutive slices compose because the second slice's first event decays from
the first slice's t_last.  Only tests/ import this module; it shares nothing
with the CUDA library.  Pinned in tests/test_slice_maps.py against the
sequential oracle (Alg. 2) on whole streams and on every split point.
"""
import math

import numpy as np

IDENT = (1.0, 0.0, -math.inf, math.inf)


def _decay(dt_us, k, b, kind):
    if kind == 2:
        return 1.0                                # Eq. 2
    if kind == 1:
        return math.exp(-k * dt_us * 1e-6)        # exponential variant (A20)
    u = 1.0 - k * dt_us * 1e-6                    # Eq. 4, reading A14
    return u ** b if u > 0.0 else 0.0


def _clamp(v, lo, hi):
    return min(max(v, lo), hi)


def mcompose(F, G):
    """F o G (G applied first), both (a, c, lo, hi) with a >= 0."""
    aF, cF, loF, hiF = F
    aG, cG, loG, hiG = G
    lo = _clamp(aF * loG + cF, loF, hiF) if loG != -math.inf else loF
    hi = _clamp(aF * hiG + cF, loF, hiF) if hiG != math.inf else hiF
    if aF == 0.0:
        lo = hi = _clamp(cF, loF, hiF)
    return (aF * aG, aF * cG + cF, lo, hi)


def mapply(G, s):
    a, c, lo, hi = G
    return _clamp(a * s + c, lo, hi)


def _event_map(dt, p, C, k, b, s_min, s_max, kind, first, unclamped):
    d = _decay(dt, k, b, kind)
    lo, hi = (-math.inf, math.inf) if (kind == 2 or unclamped) else (s_min, s_max)
    return (d, p * C if first else d * p * C, lo, hi)


def slice_maps(width, height, t, x, y, p, C=0.15, k=10.0, b=2.0, s_min=-1.5, s_max=1.5,
               decay_kind=0, decay_first=0, state_unclamped=0):
    """Dict pixel -> (n, t_first, p_first, G, t_last) over the events (arrival order)."""
    out = {}
    for i in range(len(t)):
        q = int(y[i]) * width + int(x[i])
        ti, pi = int(t[i]), int(p[i])
        if q not in out:
            out[q] = [1, ti, pi, IDENT, ti]
        else:
            m = out[q]
            g = _event_map(ti - m[4], pi, C, k, b, s_min, s_max, decay_kind, decay_first, state_unclamped)
            m[3] = mcompose(g, m[3])
            m[0] += 1
            m[4] = ti
    return {q: tuple(v) for q, v in out.items()}


def compose(A, B, C=0.15, k=10.0, b=2.0, s_min=-1.5, s_max=1.5, decay_kind=0, decay_first=0, state_unclamped=0):
    """Slice maps of A followed by B."""
    out = dict(A)
    for q, mb in B.items():
        if q not in A:
            out[q] = mb
            continue
        na, tfa, pfa, Ga, tla = A[q]
        nb, tfb, pfb, Gb, tlb = mb
        h = _event_map(tfb - tla, pfb, C, k, b, s_min, s_max, decay_kind, decay_first, state_unclamped)
        out[q] = (na + nb, tfa, pfa, mcompose(Gb, mcompose(h, Ga)), tlb)
    return out


def apply(M, S, T, C=0.15, k=10.0, b=2.0, s_min=-1.5, s_max=1.5, decay_kind=0, decay_first=0, state_unclamped=0):
    """(S, T) (flat float64 / int64 arrays, copied) after the slice."""
    S = np.array(S, np.float64).ravel().copy()
    T = np.array(T, np.int64).ravel().copy()
    lo, hi = (-math.inf, math.inf) if (decay_kind == 2 or state_unclamped) else (s_min, s_max)
    for q, (n, tf, pf, G, tl) in M.items():
        d = _decay(tf - int(T[q]), k, b, decay_kind)
        s1 = S[q] * d + pf * C if decay_first else (S[q] + pf * C) * d
        S[q] = mapply(G, _clamp(s1, lo, hi))
        T[q] = tl
    return S, T


def to_arrays(M, P):
    """Dense arrays (n, t_first, t_last, p_first, a, c, lo, hi) over P pixels (n = 0: identity)."""
    n = np.zeros(P, np.int64)
    tf = np.zeros(P, np.int64)
    tl = np.zeros(P, np.int64)
    pf = np.zeros(P, np.int64)
    G = np.tile(np.array(IDENT), (P, 1))
    for q, (nn, a_tf, a_pf, g, a_tl) in M.items():
        n[q], tf[q], tl[q], pf[q] = nn, a_tf, a_tl, a_pf
        G[q] = g
    return n, tf, tl, pf, G
