"""Search padded shared-memory layouts for the OLS exchange buffers.

The fused kernel keeps E = 16 complex samples per thread and moves a segment
between "windows" (groups of 4 index bits) through shared memory.  Element e
of thread t in window q sits at in-place index
    p = ((t >> lo) << (lo + LOGE)) | (e << lo) | (t & (2^lo - 1)),
and is stored at
    pos(p) = p + PAD1 * (p >> K1) + PAD2 * (p >> K2) + seg * STRIDE.
pos is linear over the disjoint thread / element bit fields, so every shared
memory address is (per-thread register) + (compile-time immediate).

This script finds, for every LOGN and precision, the cheapest (K1, PAD1, K2,
PAD2, STRIDE) with zero bank conflicts for every access the kernel issues:
  * J window (lo = 0): float -> 128-bit pairs (e, e+1); double -> 128-bit
  * other windows: float -> 64-bit; double -> 128-bit
Prints a C++ table consumed by csrc/olsb_fft.cuh.
"""

import itertools
import sys


def geo(logn):
    loge = min(4, logn)
    logt = logn - loge
    p = (logn + 3) // 4
    g0 = logn - 4 * (p - 1)
    los = [0] + [logn - 4 * (p - q) for q in range(1, p)]
    return loge, logt, p, g0, los


def perm(logn, q, t):
    """Geo::perm (olsb_fft.cuh): lower windows swap thread bits (lo-2, lo-1)
    with the top two thread bits so the tangent-form choice is warp-uniform."""
    loge, logt, p, g0, los = geo(logn)
    lo = los[q]
    if logn == 12 or not (q >= 1 and 2 <= lo < 7 and logt >= 7 and lo <= logt - 2):
        return t     # (not at LOGN = 12: see Geo::remap)
    a, b = lo - 2, logt - 2
    x = ((t >> a) ^ (t >> b)) & 3
    return t ^ (x << a) ^ (x << b)


def index(logn, q, e, t):
    loge, logt, p, g0, los = geo(logn)
    lo = los[q]
    t = perm(logn, q, t)
    return ((t >> lo) << (lo + loge)) | (e << lo) | (t & ((1 << lo) - 1))


def pos(p, *kp):
    """pos(p, k1, p1, k2, p2[, k3, p3]) = p + sum_i p_i * (p >> k_i)."""
    return p + sum(kp[i + 1] * (p >> kp[i]) for i in range(0, len(kp), 2))


def conflict_free(logn, segs, *args):
    *kp, stride, dbl = args
    loge, logt, npass, g0, los = geo(logn)
    T = 1 << logt
    E = 1 << loge
    nthreads = T * segs
    for q in range(npass):
        if dbl:
            width_elems, lanes_per_phase, banks_units = 1, 8, 8   # 16B units
        elif q == 0 and E >= 2:
            width_elems, lanes_per_phase, banks_units = 2, 8, 8
        else:
            width_elems, lanes_per_phase, banks_units = 1, 16, 16  # 8B units
        for e0 in range(0, E, width_elems):
            for w0 in range(0, nthreads, 32):
                for ph in range(0, 32, lanes_per_phase):
                    seen = {}
                    for lane in range(ph, ph + lanes_per_phase):
                        tid = w0 + lane
                        if tid >= nthreads:
                            continue
                        seg, t = divmod(tid, T)
                        pp = index(logn, q, e0, t)
                        a = seg * stride + pos(pp, *kp)
                        if width_elems == 2:
                            if a % 2:
                                return False
                            unit = (a // 2) % banks_units
                            key = a // 2
                        else:
                            unit = a % banks_units
                            key = a
                        if unit in seen and seen[unit] != key:
                            return False
                        seen[unit] = key
    return True


def span(logn, *kp):
    n = 1 << logn
    return pos(n - 1, *kp) + 1


def search(logn, segs, dbl, nterms=2):
    """Cheapest nterms-term padding (3 terms needed where Geo::remap swaps
    thread bits, e.g. fp32 LOGN = 11)."""
    best = None
    ks = list(range(2, logn + 1))
    pads = [0, 1, 2, 3, 4, 6, 8, 12, 16]
    for K in itertools.combinations_with_replacement(ks, nterms):
        for P in itertools.product(pads, repeat=nterms):
            kp = [v for pair in zip(K, P) for v in pair]
            sp = span(logn, *kp)
            for extra in range(0, 17, 1 if segs > 1 else 17):
                stride = sp + extra
                if dbl is False and stride % 2:
                    stride += 1
                if best is not None and stride * segs >= best[0]:
                    break
                if conflict_free(logn, segs, *kp, stride, dbl):
                    best = (stride * segs, *kp, stride)
                    break
    return best


# ---------------------------------------------------------------------------
# Per-exchange layouts (olsb_fft.cuh xpad_for): index bit b is rotated to
# address bit 0 so 128-bit accesses pair samples differing in that bit.
# `sides` = [(window, paired element bit or None for 64-bit), ...].
# ---------------------------------------------------------------------------
def rot(p, b):
    # move index bit b to address bit 0
    if b == 0: return p
    return ((p >> (b + 1)) << (b + 1)) | ((p & ((1 << b) - 1)) << 1) | ((p >> b) & 1)

def xpos(p, b, kp):
    q = rot(p, b)
    return q + sum(kp[i+1] * (q >> kp[i]) for i in range(0, len(kp), 2))

def accesses(logn, q, pb):
    """(width_elems, lanes_per_phase, units) and element groups for window q;
    pb = element bit paired in 128-bit accesses (None = 64-bit)"""
    loge, logt, npass, g0, los = geo(logn)
    E = 1 << loge
    if pb is None:
        return 1, 16, 16, [(e,) for e in range(E)]
    return 2, 8, 8, [(e, e | (1 << pb)) for e in range(E) if not (e >> pb) & 1]

def xconflict_free(logn, b, kp, sides):
    loge, logt, npass, g0, los = geo(logn)
    T = 1 << logt
    for (q, pb) in sides:
        w, lpp, bu, groups = accesses(logn, q, pb)
        for g in groups:
            for w0 in range(0, T, 32):
                for ph in range(0, 32, lpp):
                    seen = {}
                    for lane in range(ph, ph + lpp):
                        t = w0 + lane
                        if t >= T: continue
                        a = xpos(index(logn, q, g[0], t), b, kp)
                        if w == 2:
                            a2 = xpos(index(logn, q, g[1], t), b, kp)
                            if a % 2 or a2 != a + 1: return False
                            unit, key = (a // 2) % bu, a // 2
                        else:
                            unit, key = a % bu, a
                        if unit in seen and seen[unit] != key: return False
                        seen[unit] = key
    return True

def xsearch(logn, b, sides, nterms):
    best = None
    ks = range(1, logn + 1)
    pads = [0, 2, 4, 6, 8, 12, 16]
    for K in itertools.combinations(ks, nterms):
        for P in itertools.product(pads, repeat=nterms):
            kp = [v for pair in zip(K, P) for v in pair]
            span = xpos((1 << logn) - 1, b, kp) + 1
            if best and span >= best[0]: continue
            if xconflict_free(logn, b, kp, sides):
                best = (span + (span & 1), kp)
    return best

def xmain():
    for logn in (9, 10, 11, 12):
        loge, logt, npass, g0, los = geo(logn)
        if g0 < 4:   # junction batch bits overlap window 1
            bA, sidesA = los[1], [(0, los[1]), (1, 0)]
        else:
            bA, sidesA = 0, [(0, 0), (1, None)]
        bB, sidesB = los[2], [(1, None), (2, 0)]
        for name, b, sides in (("A", bA, sidesA), ("B", bB, sidesB)):
            res = None
            for nt in (1, 2, 3):
                res = xsearch(logn, b, sides, nt)
                if res:
                    break
            print(logn, name, "rotbit", b, sides, res, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "x":
        xmain()
        sys.exit(0)
    out = []
    for dbl in (False, True):
        for logn in range(2, 13):
            loge, logt, _, _, _ = geo(logn)
            T = 1 << logt
            segs = max(1, 128 // T) if not dbl else max(1, 64 // T)
            b = search(logn, segs, dbl) or search(logn, segs, dbl, 3)
            n = 1 << logn
            print(f"{'double' if dbl else 'float '} LOGN={logn:2d} segs={segs:3d} "
                  f"-> {b}  overhead {b[0] / (n * segs) - 1:.3f}", file=sys.stderr)
            out.append((dbl, logn, segs, b))
    for dbl, logn, segs, b in out:
        kp = list(b[1:-1])
        while len(kp) < 6:
            kp += [kp[-2], 0]
        print(f"  {{{int(dbl)}, {logn}, {segs}, {', '.join(map(str, kp))}, {b[-1]}}},")
