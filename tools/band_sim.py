"""Exactness simulation of the Ukkonen band cut-off for the multi-block
bit-parallel edit distance (lower blocks join late, upper blocks retire with
their deltas folded into a boundary value).  It checks, on random strings and
radii, that distances <= band come out exact and larger ones stay > band.
The cut-off was measured slower on B200 and is not in the product path
(DESIGN.md §4); this script documents the derivation.

    python tools/band_sim.py
"""
import random
M32 = 0xffffffff
def stepb(Eq, Pv, Mv, hp, hm):
    Xv = Eq | Mv
    Eq |= hm
    Xh = ((((Eq & Pv) + Pv) & M32) ^ Pv) | Eq
    Ph = Mv | (~(Xh | Pv) & M32)
    Mh = Pv & Xh
    op, om = Ph >> 31, Mh >> 31
    Ph = ((Ph << 1) & M32) | hp
    Mh = ((Mh << 1) & M32) | hm
    Pv = Mh | (~(Xv | Ph) & M32)
    Mv = Ph & Xv
    return Pv, Mv, op, om
def edit(a, b):
    m, n = len(a), len(b)
    d = list(range(m + 1))
    for j in range(1, n + 1):
        prev, d[0] = d[0], j
        for i in range(1, m + 1):
            cur = d[i]
            d[i] = min(d[i] + 1, d[i - 1] + 1, prev + (a[i - 1] != b[j - 1]))
            prev = cur
    return d[m]
def banded(a, b, band, W):
    m, n = len(a), len(b)
    peq = {}
    for c in set(a) | set(b):
        peq[c] = [0] * W
    for i, c in enumerate(a):
        peq[c][i // 32] |= 1 << (i % 32)
    P = [M32] * W; Mv = [0] * W
    wl = (m + 31) // 32
    lo_max = max(0, wl - 1); lo = 0; bval = 0
    def retire(jf):
        nonlocal lo, bval
        while lo < lo_max and 32 * (lo + 1) + band < jf:
            bval += bin(P[lo]).count('1') - bin(Mv[lo]).count('1'); lo += 1
    def char(c, nb):
        hp, hm = 1, 0
        for bb in range(W):
            if lo <= bb < nb:
                P[bb], Mv[bb], hp, hm = stepb(peq[c][bb], P[bb], Mv[bb], hp, hm)
    nfull = n // 4
    for jw in range(nfull):
        retire(4 * jw + 1)
        nb = min(W, (4 * jw + 4 + band - 1) // 32 + 1)
        for k in range(4): char(b[4 * jw + k], nb)
    rem = n & 3
    if rem:
        retire(4 * nfull + 1)
        nb = min(W, (n + band - 1) // 32 + 1)
        for k in range(rem): char(b[4 * nfull + k], nb)
    lastmask = ((1 << (m % 32)) - 1) if m % 32 else M32
    score = bval + n
    for bb in range(lo, W):
        mk = M32 if bb < wl - 1 else (lastmask if bb == wl - 1 else 0)
        score += bin(P[bb] & mk).count('1') - bin(Mv[bb] & mk).count('1')
    return score
random.seed(1)
bad = 0
for t in range(3000):
    m = random.randint(33, 128); W = (m + 31) // 32
    n = random.randint(max(0, m - 20), m + 20) if t % 2 else random.randint(1, 140)
    alpha = random.choice(["ACGT", "ab", "abcdefghij"])
    a = "".join(random.choice(alpha) for _ in range(m))
    if t % 3 == 0:
        b = list(a)
        for _ in range(random.randint(0, 12)):
            p = random.randrange(len(b) + 1)
            if random.random() < 0.5 and b: b[min(p, len(b) - 1)] = random.choice(alpha)
            else: b.insert(p, random.choice(alpha))
        b = "".join(b)[:140]
    else:
        b = "".join(random.choice(alpha) for _ in range(n))
    d = edit(a, b)
    for band in (0, 1, 3, 8, 15, 31, 40, 64, 100):
        if band >= 32 * W: continue
        s = banded(a, b, band, W)
        if (d <= band and s != d) or (d > band and s <= band):
            bad += 1
            if bad < 5: print("BAD", m, len(b), band, d, s)
print("bad", bad)
