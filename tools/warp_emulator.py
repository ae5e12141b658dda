"""Lane-level numpy emulation of k_u8_3d.cu's sweep (debug aid, not product).

Mirrors the kernel step by step -- windows, byte interleave, bit transpose,
tournament, gather, carry-save sum, histogram -- on 32 lanes x 32 bits, so a
logic error can be found without a GPU.  Usage: python tools/warp_emulator.py
"""
import os
import sys

import numpy as np

M = 0xFFFFFFFF
sys.path.insert(0, "/tmp")
from tp import dswap, transpose8, interleave  # noqa: E402


def gt(a, b):
    c = a[0] & ~b[0] & M
    for i in range(1, 8):
        c = ((a[i] & ~b[i]) | ((a[i] | (~b[i] & M)) & c)) & M
    return c


def sel(g, a, b):
    return [((g & b[i]) | (~g & M & a[i])) for i in range(8)]


def fa(a, b, c):
    return a ^ b ^ c, ((a & b) | (c & (a ^ b)))


def csa(t):
    ONE = M
    s1 = [0] * 9; c2 = [0] * 9
    for i in range(8):
        s1[i], c2[i] = fa(t[3 * i], t[3 * i + 1], t[3 * i + 2])
    s1[8], c2[8] = fa(t[24], t[25], ONE)
    s1b = [0] * 3; c2b = [0] * 3
    for i in range(3):
        s1b[i], c2b[i] = fa(s1[3 * i], s1[3 * i + 1], s1[3 * i + 2])
    bit0, c2c = fa(s1b[0], s1b[1], s1b[2])
    s2 = [0] * 4; c4 = [0] * 4
    s2[0], c4[0] = fa(c2[0], c2[1], c2[2]); s2[1], c4[1] = fa(c2[3], c2[4], c2[5])
    s2[2], c4[2] = fa(c2[6], c2[7], c2[8]); s2[3], c4[3] = fa(c2b[0], c2b[1], c2b[2])
    s2b = [0] * 2; c4b = [0] * 2
    s2b[0], c4b[0] = fa(s2[0], s2[1], s2[2]); s2b[1], c4b[1] = fa(s2[3], c2c, ONE)
    bit1 = s2b[0] ^ s2b[1]; c4c = s2b[0] & s2b[1]
    s4 = [0] * 2; c8 = [0] * 2
    s4[0], c8[0] = fa(c4[0], c4[1], c4[2]); s4[1], c8[1] = fa(c4[3], c4b[0], c4b[1])
    bit2, c8c = fa(s4[0], s4[1], c4c)
    bit3 = (~(c8[0] ^ c8[1] ^ c8c)) & M
    return bit0, bit1, bit2, bit3


def emulate(img):
    W0, W1, W2 = img.shape
    Gy, Gz = (W1 + 29) // 30, (W2 + 29) // 30
    hist = np.zeros(256, np.int64)
    for gy in range(Gy):
        for gz in range(Gz):
            ys, ye = gy * W1 // Gy, (gy + 1) * W1 // Gy
            zs, ze = gz * W2 // Gz, (gz + 1) * W2 // Gz
            z0 = zs - 1
            nz = ze - zs
            own = ((1 << (nz + 1)) - 1) & ~1
            P = None
            xc = None
            for X in range(-1, W0 + 1):
                lanes = []
                for lane in range(32):
                    y = ys - 1 + lane
                    by = []
                    for p in range(32):
                        z = z0 + p
                        inimg = 0 <= X < W0 and 0 <= y < W1 and 0 <= z < W2
                        by.append(int(img[X, y, z]) if inimg else 255)
                    a = [by[4 * j] | by[4 * j + 1] << 8 | by[4 * j + 2] << 16 | by[4 * j + 3] << 24 for j in range(8)]
                    wv = interleave(a)
                    C = transpose8(wv)
                    lanes.append((y, wv, C))
                N = [dict() for _ in range(32)]
                for lane in range(32):
                    y, wv, C = lanes[lane]
                    Cz = [c >> 1 for c in C]
                    g = gt(C, Cz)
                    if z0 < 0:
                        g |= 1
                    mz = sel(g, C, Cz)
                    N[lane].update(C=C, wv=wv, mz=mz, gz=g, y=y)
                for lane in range(32):
                    C = N[lane]["C"]
                    Cy = N[min(lane + 1, 31)]["C"] if lane < 31 else C
                    gy_ = gt(C, Cy)
                    if N[lane]["y"] < 0:
                        gy_ = M
                    N[lane]["my"] = sel(gy_, C, Cy)
                    N[lane]["gy"] = gy_
                    mz = N[lane]["mz"]
                    mzy = N[lane + 1]["mz"] if lane < 31 else mz
                    gyz = gt(mz, mzy)
                    if N[lane]["y"] < 0:
                        gyz = M
                    N[lane]["myz"] = sel(gyz, mz, mzy)
                    N[lane]["gyz"] = gyz
                for lane in range(32):
                    n = N[lane]
                    n["bz"], n["by"], n["byz"] = ~n["gz"] & M, ~n["gy"] & M, ~n["gyz"] & M
                if P is not None:
                    cur = []
                    for lane in range(32):
                        pl, n = P[lane], N[lane]
                        bx = ~gt(pl["C"], n["C"]) & M
                        bxz = ~gt(pl["mz"], n["mz"]) & M
                        bxy = ~gt(pl["my"], n["my"]) & M
                        b8 = ~gt(pl["myz"], n["myz"]) & M
                        if X - 1 < 0:
                            bx = bxz = bxy = b8 = 0
                        cur.append(dict(bx=bx, bxz=bxz, bxy=bxy, b8=b8))
                    for lane in range(32):
                        cur[lane]["bxyu"] = cur[lane - 1]["bxy"] if lane > 0 else cur[0]["bxy"]
                        cur[lane]["b8u"] = cur[lane - 1]["b8"] if lane > 0 else cur[0]["b8"]
                    if xc is not None and 0 <= X - 1 < W0:
                        for lane in range(32):
                            pl = P[lane]
                            up = P[lane - 1] if lane > 0 else P[0]
                            c, q = cur[lane], xc[lane]
                            byu, byzu = up["by"], up["byz"]
                            Z0 = pl["bz"]; Z1 = ~(pl["bz"] << 1) & M
                            Yf0 = pl["by"]; Yf1 = ~byu & M
                            Y00 = pl["byz"]; Y01 = (pl["byz"] << 1) & M; Y10 = ~byzu & M; Y11 = ~(byzu << 1) & M
                            I00, I01, I10, I11 = Z0 & Y00, Z1 & Y01, Z0 & Y10, Z1 & Y11
                            n_ = lambda v: ~v & M
                            t = [Z0, Z1, Yf0, Yf1, c["bx"], n_(q["bx"]),
                                 n_(I00), n_(I01), n_(I10), n_(I11),
                                 n_(Z0 & c["bxz"]), n_(Z1 & ((c["bxz"] << 1) & M)),
                                 n_(Z0 & n_(q["bxz"])), n_(Z1 & n_((q["bxz"] << 1) & M)),
                                 n_(Yf0 & c["bxy"]), n_(Yf1 & c["bxyu"]),
                                 n_(Yf0 & n_(q["bxy"])), n_(Yf1 & n_(q["bxyu"])),
                                 I00 & c["b8"], I01 & ((c["b8"] << 1) & M), I10 & c["b8u"], I11 & ((c["b8u"] << 1) & M),
                                 I00 & n_(q["b8"]), I01 & n_((q["b8"] << 1) & M), I10 & n_(q["b8u"]),
                                 I11 & n_((q["b8u"] << 1) & M)]
                            b0, b1, b2, b3 = csa(t)
                            if not (1 <= lane <= ye - ys):
                                continue
                            for p in range(1, 31):
                                if not (own >> p) & 1:
                                    continue
                                v = ((b0 >> p) & 1) | ((b1 >> p) & 1) << 1 | ((b2 >> p) & 1) << 2 | ((b3 >> p) & 1) << 3
                                r, b = p % 8, p // 8
                                val = (pl["wv"][r] >> (8 * b)) & 255
                                hist[val] += v - 8
                    xc = cur
                P = N
    return hist


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    rng = np.random.default_rng(0)
    shape = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (3, 30, 32)
    img = rng.integers(0, 256, shape).astype(np.uint8)
    h = emulate(img)
    v, c = oracle.vcec(img)
    got = h[v.astype(np.int64)]
    print("emulator == oracle:", np.array_equal(got, c))
    print(got[:10], c[:10])
