"""Exact-math pins for the DSI latency models (test infrastructure, Python fractions).

Nothing here is imported by the product or by the oracle.  These are derived
closed forms that pin both of them from outside:

* Segments.  The rejected positions z_1 < ... < z_{m-1} among 1..N-1 cut a trial
  into segments g_s = z_s - z_{s-1} (z_0 = 0, z_m = N).  Every segment starts with
  all servers free (a rejection terminates every thread, Alg. 1 lines 8/10,
  P:128-130), so its DSI cost depends on g only.
* DSI segment cost (Alg. 1 P:112-142 + App. D, R1-R10):
  thread b (b = 0 on the committed prefix, b >= 1 after b*k drafts) is requested
  at b*k*t_d; with SP FIFO servers and equal service t_t it starts at
  S(b) = max(b*k*t_d, S(b-SP) + t_t) = max(b k t_d, (b mod SP) k t_d + floor(b/SP) t_t);
  position j of a segment is settled by thread ceil((j-1)/k), hence
  C(g) = t_t + S(ceil((g-1)/k)).
* SI: an iteration ends at min(next zero, start+k+1), so
  I = sum_s ceil(g_s/(k+1)) and L_SI = I (k t_d + t_t).
* Expected number of segments of length g (i.i.d. Bernoulli(a)):
  h(g) = (1-a) a^(g-1) [2 + (1-a)(N-1-g)] for g <= N-1, h(N) = a^(N-1).
"""
from __future__ import annotations

from fractions import Fraction
from itertools import product


def segments(A, N):
    """Segment lengths of an indicator vector A[0..N-2] (A[p-1] = A_p)."""
    out, last = [], 0
    for p in range(1, N):
        if A[p - 1] == 0:
            out.append(p - last)
            last = p
    out.append(N - last)
    return out


def S(b, k, t_d, t_t, sp):
    return max(b * k * t_d, (b % sp) * k * t_d + (b // sp) * t_t)


def C(g, k, t_d, t_t, sp):
    b = -(-(g - 1) // k)
    return t_t + S(b, k, t_d, t_t, sp)


def closed_form(A, N, k, t_d, t_t, sp):
    """Per-trial (acc, m, I, L_SI, L_DSI, L_non) from the closed form."""
    gs = segments(A, N)
    iters = sum(-(-g // (k + 1)) for g in gs)
    return {"acc": sum(A[: N - 1]), "m": len(gs), "iters": iters,
            "si": iters * (k * t_d + t_t), "dsi": sum(C(g, k, t_d, t_t, sp) for g in gs),
            "nonsi": N * t_t}


def h(g, N, a):
    a = Fraction(a)
    if g == N:
        return a ** (N - 1)
    return (1 - a) * a ** (g - 1) * (2 + (1 - a) * (N - 1 - g))


def expectations(N, k, t_d, t_t, sp, a):
    """Exact E[L_DSI], E[I], E[L_SI], E[m], E[acc] as Fractions."""
    a = Fraction(a)
    e_dsi = sum(h(g, N, a) * C(g, k, t_d, t_t, sp) for g in range(1, N + 1))
    e_i = sum(h(g, N, a) * (-(-g // (k + 1))) for g in range(1, N + 1))
    return {"dsi": e_dsi, "iters": e_i, "si": e_i * (k * t_d + t_t),
            "m": 1 + (1 - a) * (N - 1), "acc": a * (N - 1), "nonsi": Fraction(N * t_t)}


def enumerate_expectations(N, a, per_pattern):
    """E[f] by brute force over all 2^(N-1) patterns with weights a^acc (1-a)^(N-1-acc).

    per_pattern(A) -> dict of numbers; returns dict of Fractions."""
    a = Fraction(a)
    tot = {}
    for A in product((0, 1), repeat=N - 1):
        acc = sum(A)
        w = a ** acc * (1 - a) ** (N - 1 - acc)
        for key, v in per_pattern(list(A)).items():
            tot[key] = tot.get(key, Fraction(0)) + w * v
    return tot


def pattern_index(A):
    """Trial index whose bits are the indicators (enumeration mode: A_p = bit p-1)."""
    return sum(int(v) << i for i, v in enumerate(A))


def expectations_grid_f64(N, t_t, t_ds, ks, sp, ps, fresh=False):
    """Exact E[L_SI], E[L_DSI] (float64) for every (p, t_d, k) of a grid: the same h(g)
    and C(g) (or, fresh=True, C_fresh(g)) formulas as above, vectorised with numpy.
    Shapes (len(ps), len(t_ds), len(ks))."""
    import numpy as np
    g = np.arange(1, N + 1, dtype=np.float64)
    ps = np.asarray(ps, dtype=np.float64)
    H = np.empty((ps.size, N))
    for i, p in enumerate(ps):
        h = (1 - p) * p ** (g - 1) * (2 + (1 - p) * (N - 1 - g))
        h[-1] = p ** (N - 1)
        H[i] = h
    ks = np.asarray(ks, dtype=np.int64)
    t_ds = np.asarray(t_ds, dtype=np.int64)
    gi = np.arange(1, N + 1, dtype=np.int64)
    b = -(-(gi[None, :] - 1) // ks[:, None])                    # (k, g)
    iters = -(-gi[None, :] // (ks[:, None] + 1))                # (k, g)
    KD = ks[None, :, None] * t_ds[:, None, None]                # (t_d, k, 1)
    S = np.maximum(b[None] * KD, (b[None] % sp) * KD + (b[None] // sp) * t_t)
    C = (t_t + S).astype(np.float64)                            # (t_d, k, g)
    if fresh:  # C_fresh where k t_d > t_t (block b, offset j; see C_fresh)
        j = gi[None, :] - 1 - (b - 1) * ks[:, None]             # (k, g)
        TD = t_ds[:, None, None]
        Cf = t_t + (b[None] - 1) * KD + np.minimum(KD, t_t * (-(-(j[None] * TD) // t_t)))
        act = (KD > t_t) & (gi[None, None, :] >= 2)
        C = np.where(act, Cf, C).astype(np.float64)
    e_dsi = np.einsum("pg,dkg->pdk", H, C)
    e_i = np.einsum("pg,kg->pk", H, iters.astype(np.float64))   # (p, k)
    e_si = e_i[:, None, :] * (KD[None, :, :, 0] + t_t)
    return e_si, e_dsi


def first_segment_costs(N, k, t_d, t_t, sp, t_t1, t_d1):
    """TTFT variant: cost C1(g) of a FIRST segment of length g, by a plain FIFO
    multi-server schedule written independently of the oracle: thread 0 (the target's
    first forward) is requested at 0 and serves t_t1; thread b >= 1 is requested when
    its k drafts are done, at t_d1 + (b k - 1) t_d, and serves t_t; positions settle in
    order, so the segment ends at max(f_0..f_b(g)), b(g) = ceil((g-1)/k)."""
    import heapq
    B = -(-(N - 1) // k) if N > 1 else 0
    free = [0] * sp
    heapq.heapify(free)
    f = []
    for b in range(B + 1):
        r = 0 if b == 0 else t_d1 + (b * k - 1) * t_d
        start = max(r, heapq.heappop(free))
        end = start + (t_t1 if b == 0 else t_t)
        heapq.heappush(free, end)
        f.append(end)
    out = {}
    for g in range(1, N + 1):
        b = -(-(g - 1) // k)
        out[g] = max(f[: b + 1])
    return out


def expectations_ttft(N, k, t_d, t_t, sp, a, t_t1, t_d1):
    """Exact E[L_DSI], E[L_SI], L_non with first-forward costs: later segments keep C(g);
    the first segment (length g with probability a^(g-1)(1-a), or a^(N-1) for g = N)
    costs C1(g); SI's first iteration pays (t_d1 - t_d) + (t_t1 - t_t) more."""
    a = Fraction(a)
    base = expectations(N, k, t_d, t_t, sp, a)
    c1 = first_segment_costs(N, k, t_d, t_t, sp, t_t1, t_d1)
    extra = Fraction(0)
    for g in range(1, N + 1):
        pg = a ** (N - 1) if g == N else a ** (g - 1) * (1 - a)
        extra += pg * (c1[g] - C(g, k, t_d, t_t, sp))
    return {"dsi": base["dsi"] + extra, "si": base["si"] + (t_d1 - t_d) + (t_t1 - t_t),
            "nonsi": Fraction(t_t1 + (N - 1) * t_t), "iters": base["iters"]}


def si_tokens_per_iteration(a, k):
    """E[n+1] = (1 - a^(k+1)) / (1 - a): truncated geometric."""
    a = Fraction(a)
    if a == 1:
        return Fraction(k + 1)
    return (1 - a ** (k + 1)) / (1 - a)


def C_fresh(g, k, t_d, t_t, sp):
    """Fresh-verifier variant (R24), derived by hand from the
    reading, not from the oracle.  If k t_d <= t_t a fresh forward never finishes sooner
    than the regular thread (S(b+1) - S(b) <= max(k t_d, t_t) = t_t), so C_fresh = C.
    Otherwise no task ever queues (requests are k t_d > t_t apart) and thread b ends at
    F_b = b k t_d + t_t; inside block b (offsets j = 1..k after position (b-1)k + 1,
    reached at F_{b-1}) fresh forward i >= 0 starts at F_{b-1} + i t_t while
    (i+1) t_t < k t_d and settles offsets up to floor((i+1) t_t / t_d), so offset j
    settles at F_{b-1} + min(k t_d, t_t ceil(j t_d / t_t))."""
    kd = k * t_d
    if g == 1 or kd <= t_t:
        return C(g, k, t_d, t_t, sp)
    b = -(-(g - 1) // k)
    j = g - 1 - (b - 1) * k
    return t_t + (b - 1) * kd + min(kd, t_t * (-(-(j * t_d) // t_t)))


def closed_form_fresh(A, N, k, t_d, t_t, sp):
    out = closed_form(A, N, k, t_d, t_t, sp)
    out["dsi"] = sum(C_fresh(g, k, t_d, t_t, sp) for g in segments(A, N))
    return out


def expectations_fresh(N, k, t_d, t_t, sp, a):
    a = Fraction(a)
    out = expectations(N, k, t_d, t_t, sp, a)
    out["dsi"] = sum(h(g, N, a) * C_fresh(g, k, t_d, t_t, sp) for g in range(1, N + 1))
    return out


def moments_dp(N, a, cost):
    """Exact (E[L], E[L^2]) of L = sum_s cost(g_s) by a renewal recursion over the positions of
    the zeros (written independently of h(g) and of any enumeration): z = 0 is the start; from
    a zero at z the next zero is at z' <= N-1 with probability a^(z'-z-1) (1-a), and with
    probability a^(N-1-z) there is none and the final segment ends at N.  Carries
    P_z = P(zero at z), M1_z = E[partial L; zero at z], M2_z = E[partial L^2; zero at z]."""
    a = Fraction(a)
    P = [Fraction(0)] * N
    M1 = [Fraction(0)] * N
    M2 = [Fraction(0)] * N
    P[0] = Fraction(1)
    e1 = e2 = Fraction(0)
    for z in range(N):  # P, M1, M2 at z are final once every z0 < z has been pushed
        if P[z] == 0 and M1[z] == 0:
            continue
        for z2 in range(z + 1, N):
            w = a ** (z2 - z - 1) * (1 - a)
            c = cost(z2 - z)
            P[z2] += w * P[z]
            M1[z2] += w * (M1[z] + c * P[z])
            M2[z2] += w * (M2[z] + 2 * c * M1[z] + c * c * P[z])
        w = a ** (N - 1 - z)
        c = cost(N - z)
        e1 += w * (M1[z] + c * P[z])
        e2 += w * (M2[z] + 2 * c * M1[z] + c * c * P[z])
    return e1, e2


def moments_dsi_si(N, k, t_d, t_t, sp, a, fresh=False):
    """Exact (E, E^2) of L_DSI and L_SI: L_DSI = sum C(g) (or C_fresh), L_SI = (k t_d + t_t)
    sum ceil(g/(k+1))."""
    cd = (lambda g: C_fresh(g, k, t_d, t_t, sp)) if fresh else (lambda g: C(g, k, t_d, t_t, sp))
    si_cost = k * t_d + t_t
    return {"dsi": moments_dp(N, a, cd),
            "si": moments_dp(N, a, lambda g: si_cost * (-(-g // (k + 1))))}
