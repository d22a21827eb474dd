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


def index(logn, q, e, t):
    loge, logt, p, g0, los = geo(logn)
    lo = los[q]
    return ((t >> lo) << (lo + loge)) | (e << lo) | (t & ((1 << lo) - 1))


def pos(p, k1, p1, k2, p2):
    return p + p1 * (p >> k1) + p2 * (p >> k2)


def conflict_free(logn, segs, k1, p1, k2, p2, stride, dbl):
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
                        a = seg * stride + pos(pp, k1, p1, k2, p2)
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


def span(logn, k1, p1, k2, p2):
    n = 1 << logn
    return pos(n - 1, k1, p1, k2, p2) + 1


def search(logn, segs, dbl):
    best = None
    ks = list(range(2, logn + 1))
    pads = [0, 1, 2, 4, 8, 16]
    for k1, k2 in itertools.product(ks, ks):
        if k2 < k1:
            continue
        for p1, p2 in itertools.product(pads, pads):
            if k1 == k2 and p2:
                continue
            sp = span(logn, k1, p1, k2, p2)
            for extra in range(0, 17, 1 if segs > 1 else 17):
                stride = sp + extra
                if dbl is False and stride % 2:
                    continue
                if conflict_free(logn, segs, k1, p1, k2, p2, stride, dbl):
                    cost = stride * segs
                    if best is None or cost < best[0]:
                        best = (cost, k1, p1, k2, p2, stride)
                    break
    return best


if __name__ == "__main__":
    out = []
    for dbl in (False, True):
        for logn in range(2, 13):
            loge, logt, _, _, _ = geo(logn)
            T = 1 << logt
            segs = max(1, 128 // T) if not dbl else max(1, 64 // T)
            b = search(logn, segs, dbl)
            n = 1 << logn
            print(f"{'double' if dbl else 'float '} LOGN={logn:2d} segs={segs:3d} "
                  f"-> {b}  overhead {b[0] / (n * segs) - 1:.3f}", file=sys.stderr)
            out.append((dbl, logn, segs, b))
    for dbl, logn, segs, b in out:
        cost, k1, p1, k2, p2, stride = b
        print(f"  {{{int(dbl)}, {logn}, {segs}, {k1}, {p1}, {k2}, {p2}, {stride}}},")
