"""Dense numpy model of the tournament formulation used by the bit-sliced
3D kernel (k_u8_3d.cu).  Not product code: it validates the algebra
(block winners -> per-voxel change) against the oracle on small volumes.

For each anchor p the kernel computes "lower side wins" bits:
  bz  = v(p) <= v(p+z)            mz  = winner value of the z-pair
  by  = v(p) <= v(p+y)            my  = winner value of the y-pair
  byz = mz(p) <= mz(p+y)          myz = winner value of the yz 4-block
  bx  = v(p) <= v(p+x)
  bxz = mz(p) <= mz(p+x)          (xz 4-block)
  bxy = my(p) <= my(p+x)          (xy 4-block)
  b8  = myz(p) <= myz(p+x)        (2x2x2 block)
Ties go to the lower (earlier in row-major order) side, which is exactly the
reference's strict/non-strict rule (kernel.hpp:21-27).  A voxel's change is
 -1 + #2-blocks it wins - #4-blocks it wins + #8-blocks it wins
(kernel.hpp:99-137 counts the same faces).
"""
import numpy as np

S = 1 << 20  # sentinel, larger than any value


def model_changes(img):
    img = np.asarray(img).astype(np.int64)
    X, Y, Z = img.shape
    # pad with sentinel on all sides: index i -> i+1
    V = np.full((X + 2, Y + 2, Z + 2), S, np.int64)
    V[1:-1, 1:-1, 1:-1] = img

    def sh(a, dx, dy, dz, fill):
        out = np.full_like(a, fill)
        sx = slice(max(0, -dx), a.shape[0] - max(0, dx))
        sy = slice(max(0, -dy), a.shape[1] - max(0, dy))
        sz = slice(max(0, -dz), a.shape[2] - max(0, dz))
        tx = slice(max(0, dx), a.shape[0] - max(0, -dx))
        ty = slice(max(0, dy), a.shape[1] - max(0, -dy))
        tz = slice(max(0, dz), a.shape[2] - max(0, -dz))
        out[sx, sy, sz] = a[tx, ty, tz]
        return out

    inside = np.zeros(V.shape, bool)
    inside[1:-1, 1:-1, 1:-1] = True
    # a sentinel never wins as the lower side
    bz = (V <= sh(V, 0, 0, 1, S)) & inside_or(V, 0)
    mz = np.where(bz, V, sh(V, 0, 0, 1, S))
    by = (V <= sh(V, 0, 1, 0, S)) & (V < S)
    my = np.where(by, V, sh(V, 0, 1, 0, S))
    mzy = sh(mz, 0, 1, 0, S)
    byz = (mz <= mzy) & (mz < S)
    myz = np.where(byz, mz, mzy)
    bx = (V <= sh(V, 1, 0, 0, S)) & (V < S)
    bxz = (mz <= sh(mz, 1, 0, 0, S)) & (mz < S)
    bxy = (my <= sh(my, 1, 0, 0, S)) & (my < S)
    b8 = (myz <= sh(myz, 1, 0, 0, S)) & (myz < S)

    def at(a, dx, dy, dz):  # value at v - (dx,dy,dz)
        return sh(a, -dx, -dy, -dz, 0).astype(np.int64)

    n = lambda a: 1 - a
    bz_, by_, byz_, bx_, bxz_, bxy_, b8_ = [a.astype(np.int64) for a in (bz, by, byz, bx, bxz, bxy, b8)]
    Z = [bz_, n(at(bz_, 0, 0, 1))]
    Yp = [by_, n(at(by_, 0, 1, 0))]
    Xf = [bx_, n(at(bx_, 1, 0, 0))]
    ch = -1 + sum(Z) + sum(Yp) + sum(Xf)
    for c in (0, 1):
        for b in (0, 1):
            ybc = at(byz_, 0, 0, c) if b == 0 else n(at(byz_, 0, 1, c))
            I = Z[c] * ybc
            ch -= I
            for a in (0, 1):
                w = at(b8_, 0, b, c) if a == 0 else n(at(b8_, 1, b, c))
                ch += I * w
        for a in (0, 1):
            xac = at(bxz_, 0, 0, c) if a == 0 else n(at(bxz_, 1, 0, c))
            ch -= Z[c] * xac
    for b in (0, 1):
        for a in (0, 1):
            xab = at(bxy_, 0, b, 0) if a == 0 else n(at(bxy_, 1, b, 0))
            ch -= Yp[b] * xab
    return ch[1:-1, 1:-1, 1:-1]


def inside_or(V, _):
    return V < S


if __name__ == "__main__":
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    rng = np.random.default_rng(0)
    for it in range(300):
        shp = tuple(rng.integers(1, 7, 3))
        hi = int(rng.choice([2, 4, 8, 256]))
        img = rng.integers(0, hi, shp).astype(np.uint8)
        want = oracle.changes(img)
        got = model_changes(img)
        assert np.array_equal(want.reshape(got.shape), got), (shp, hi)
    print("tournament model == oracle changes on 300 random volumes")


def model_changes_255(img):
    """Same, but the collar holds 255 (what the kernel's planes hold) and only
    the comparisons whose LOWER operand lies on the -1 collar are forced."""
    img = np.asarray(img).astype(np.int64)
    X, Y, Z = img.shape
    V = np.full((X + 2, Y + 2, Z + 2), 255, np.int64)
    V[1:-1, 1:-1, 1:-1] = img

    def nxt(a, ax):
        out = np.full_like(a, 255)
        sl = [slice(None)] * 3
        sl2 = [slice(None)] * 3
        sl[ax] = slice(0, -1)
        sl2[ax] = slice(1, None)
        out[tuple(sl)] = a[tuple(sl2)]
        return out

    lo = np.zeros(V.shape, bool)  # x=-1 collar plane
    bz = V <= nxt(V, 2); bz[:, :, 0] = False
    mz = np.where(bz, V, nxt(V, 2))
    by = V <= nxt(V, 1); by[:, 0, :] = False
    my = np.where(by, V, nxt(V, 1))
    byz = mz <= nxt(mz, 1); byz[:, 0, :] = False
    myz = np.where(byz, mz, nxt(mz, 1))
    bx = V <= nxt(V, 0); bxz = mz <= nxt(mz, 0); bxy = my <= nxt(my, 0); b8 = myz <= nxt(myz, 0)
    for a in (bx, bxz, bxy, b8):
        a[0, :, :] = False
    bz_, by_, byz_, bx_, bxz_, bxy_, b8_ = [a.astype(np.int64) for a in (bz, by, byz, bx, bxz, bxy, b8)]

    def at(a, dx, dy, dz):
        out = np.zeros_like(a)
        out[dx:, dy:, dz:] = a[:a.shape[0] - dx, :a.shape[1] - dy, :a.shape[2] - dz]
        return out
    n = lambda a: 1 - a
    Zs = [bz_, n(at(bz_, 0, 0, 1))]
    Yp = [by_, n(at(by_, 0, 1, 0))]
    ch = -1 + sum(Zs) + sum(Yp) + bx_ + n(at(bx_, 1, 0, 0))
    for c in (0, 1):
        for b in (0, 1):
            ybc = at(byz_, 0, 0, c) if b == 0 else n(at(byz_, 0, 1, c))
            I = Zs[c] * ybc
            ch -= I
            for a in (0, 1):
                ch += I * (at(b8_, 0, b, c) if a == 0 else n(at(b8_, 1, b, c)))
        for a in (0, 1):
            ch -= Zs[c] * (at(bxz_, 0, 0, c) if a == 0 else n(at(bxz_, 1, 0, c)))
    for b in (0, 1):
        for a in (0, 1):
            ch -= Yp[b] * (at(bxy_, 0, b, 0) if a == 0 else n(at(bxy_, 1, b, 0)))
    return ch[1:-1, 1:-1, 1:-1]


def check_255(n=300):
    import oracle
    rng = np.random.default_rng(1)
    for it in range(n):
        shp = tuple(rng.integers(1, 7, 3))
        hi = int(rng.choice([2, 4, 256]))
        img = rng.integers(256 - hi, 256, shp).astype(np.uint8)  # values near 255
        want = oracle.changes(img)
        got = model_changes_255(img)
        assert np.array_equal(want.reshape(got.shape), got), (shp, hi)
    print("255-collar model == oracle changes on", n, "volumes")
