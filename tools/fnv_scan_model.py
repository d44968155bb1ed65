"""Executable model of the device FNV-1a-64 scan (lzk_fnv_kernel), used to
check the bit-plane algorithm before/while writing CUDA. Not shipped.

FNV-1a-64 step: h' = (h ^ b) * P, P = 0x100000001b3 (checksum.hpp:17-24).
Low byte l = h & 0xff evolves alone: l' = 0xb3 * (l ^ b) mod 256 (SURVEY
Appendix C). Because the low byte of ANY state with the right low byte
follows the true trajectory, running plain FNV from the 64-bit value `l`
gives acc = P^n * l + S, where S is the true segment contribution:
    h_end = P^n * h_start + (acc - P^n * l).
So a warp only needs the low byte at the start of every lane's 32-byte
segment; those come from a bit-sliced scan over the 8 planes of l (each
plane is a prefix-XOR once the lower planes are known, because
multiplication by an odd constant is a T-function).
"""
import random

P = 0x100000001B3
M64 = (1 << 64) - 1
BASIS = 0xCBF29CE484222325


def fnv(data, h=BASIS):
    for b in data:
        h = ((h ^ b) * P) & M64
    return h


def planes_of(seg):
    """32 bytes -> 8 plane words, bit p of plane i = bit i of byte p."""
    return [sum(((seg[p] >> i) & 1) << p for p in range(len(seg))) for i in range(8)]


def maj(a, b, c):
    return (a & b) | (a & c) | (b & c)


def warp_chunk(chunk, lchunk):
    """One 1 KiB chunk (32 lanes x 32 B) -> per-lane start low bytes, and the
    chunk's outgoing low byte. Mirrors the CUDA control flow (ballot scan)."""
    nl = 32
    segs = [chunk[32 * j:32 * j + 32] for j in range(nl)]
    Bs = [planes_of(s) for s in segs]
    lstart = [0] * nl
    carry = [(lchunk >> i) & 1 for i in range(8)]
    lane_X = [[0] * 8 for _ in range(nl)]
    for i in range(8):
        ps = []
        for j in range(nl):
            B = Bs[j]
            X = lane_X[j]
            e = plane_e(i, B, X)
            p = e
            for sh in (1, 2, 4, 8, 16):
                p ^= (p << sh) & 0xFFFFFFFF
            ps.append(p)
        bal = sum(((ps[j] >> 31) & 1) << j for j in range(nl))
        for j in range(nl):
            cin = (bin(bal & ((1 << j) - 1)).count("1") + carry[i]) & 1
            l_word = ((ps[j] << 1) & 0xFFFFFFFF) ^ (0xFFFFFFFF if cin else 0)
            lane_X[j][i] = l_word ^ Bs[j][i]
            lstart[j] |= cin << i
        carry[i] ^= bin(bal).count("1") & 1
    lout = sum(carry[i] << i for i in range(8))
    return lstart, lout


def plane_e(i, B, X):
    """e_i = b_i ^ g_i(x_<i) — the bit-sliced column adder of y = 179 * x (mod 256)."""
    if i == 0:
        return B[0]
    if i == 1:
        return B[1] ^ X[0]
    c2 = X[1] & X[0]
    if i == 2:
        return B[2] ^ X[1] ^ c2
    c3 = maj(X[2], X[1], c2)
    if i == 3:
        return B[3] ^ X[2] ^ c3
    c4 = maj(X[3], X[2], c3)
    if i == 4:
        return B[4] ^ X[3] ^ X[0] ^ c4
    s = X[4] ^ X[3] ^ X[0]
    k1 = maj(X[4], X[3], X[0])
    k2 = s & c4
    if i == 5:
        return B[5] ^ X[4] ^ X[1] ^ X[0] ^ k1 ^ k2
    s1 = X[5] ^ X[4] ^ X[1]
    m1 = maj(X[5], X[4], X[1])
    s2 = X[0] ^ k1 ^ k2
    m2 = maj(X[0], k1, k2)
    m3 = s1 & s2
    if i == 6:
        return B[6] ^ X[5] ^ X[2] ^ X[1] ^ m1 ^ m2 ^ m3
    t1 = X[6] ^ X[5] ^ X[2]
    n1 = maj(X[6], X[5], X[2])
    t2 = X[1] ^ m1 ^ m2
    n2 = maj(X[1], m1, m2)
    n3 = maj(m3, t1, t2)
    return B[7] ^ X[6] ^ X[3] ^ X[2] ^ X[0] ^ n1 ^ n2 ^ n3


def fnv_model(data, h0=BASIS):
    n = len(data)
    full = n // 1024
    h = h0
    l = h0 & 0xFF
    for c in range(full):
        chunk = data[1024 * c:1024 * c + 1024]
        lstart, lout = warp_chunk(chunk, l)
        S = 0
        for j in range(32):
            acc = lstart[j]
            acc = fnv(chunk[32 * j:32 * j + 32], acc)
            seg = (acc - pow(P, 32, 1 << 64) * lstart[j]) & M64
            S = (S + seg * pow(P, 32 * (31 - j), 1 << 64)) & M64
        h = (pow(P, 1024, 1 << 64) * h + S) & M64
        assert h & 0xFF == lout, (h & 0xFF, lout)
        l = lout
    return fnv(data[1024 * full:], h)


if __name__ == "__main__":
    rng = random.Random(7)
    # low-byte recurrence sanity
    for _ in range(2000):
        h, b = rng.getrandbits(64), rng.getrandbits(8)
        assert (((h ^ b) * P) & 0xFF) == ((0xB3 * ((h & 0xFF) ^ b)) & 0xFF)
    for n in (0, 1, 31, 1023, 1024, 1025, 3000, 4096, 5000):
        d = bytes(rng.getrandbits(8) for _ in range(n))
        h0 = rng.getrandbits(64) if n % 2 else BASIS
        assert fnv_model(d, h0) == fnv(d, h0), n
    print("model ok")


def segment_parity(data, lin, planes):
    """Per-segment plane parities as the pass kernels compute them: bit i of
    the low byte at the segment end, evaluated with the carry-in bits < i
    right and bit i forced to 0 (T-function: bits <= i only see bits <= i)."""
    par = 0
    for i in range(planes):
        l = lin & ((1 << i) - 1)
        for b in data:
            l = (0xB3 * (l ^ b)) & 0xFF
        par |= ((l >> i) & 1) << i
    return par


def segmented(data, h0, seglen):
    """Multi-pass long-chain scheme (lzk_fnv.cu segmented path)."""
    segs = [data[k:k + seglen] for k in range(0, len(data), seglen)] or [b""]
    l0 = h0 & 0xFF
    par = [segment_parity(s, 0, 0) for s in segs]
    for i in range(8):  # pass i: carry-in bits < i from the parity prefix
        for k, s in enumerate(segs[:-1]):
            lin = l0
            for q in par[:k]:
                lin ^= q
            par[k] |= ((segment_parity(s, lin, i + 1) >> i) & 1) << i
    h = h0
    for k, s in enumerate(segs):  # final pass + combine
        lin = l0
        for q in par[:k]:
            lin ^= q
        assert lin == h & 0xFF
        acc = fnv(s, lin)
        h = (pow(P, len(s), 1 << 64) * h + acc - pow(P, len(s), 1 << 64) * lin) & M64
    return h


if __name__ == "__main__":
    rng = random.Random(9)
    for n, sl in ((5000, 1024), (4097, 2048), (3000, 1000), (64, 16)):
        d = bytes(rng.getrandbits(8) for _ in range(n))
        h0 = rng.getrandbits(64)
        assert segmented(d, h0, sl) == fnv(d, h0), (n, sl)
    print("segmented ok")


def dual_chunk(chunk, carry, K):
    """Bit-sliced model of scan_dual<K> (one 1 KiB window): planes 0..2K with
    the carry-ins in `carry`, then plane 2K+1's parity for x_{2K} and for its
    complement (incoming bit 2K = 0 / 1). Returns (carry, alt_parity)."""
    nl = 32
    Bs = [planes_of(chunk[32 * j:32 * j + 32]) for j in range(nl)]
    X = [[0] * 8 for _ in range(nl)]
    carry = list(carry)

    def pref(e):
        p = e
        for sh in (1, 2, 4, 8, 16):
            p ^= (p << sh) & 0xFFFFFFFF
        return p

    for i in range(2 * K + 1):
        ps = [pref(plane_e(i, Bs[j], X[j])) for j in range(nl)]
        bal = sum(((ps[j] >> 31) & 1) << j for j in range(nl))
        for j in range(nl):
            cin = (bin(bal & ((1 << j) - 1)).count("1") + carry[i]) & 1
            X[j][i] = ((ps[j] << 1) & 0xFFFFFFFF) ^ (0xFFFFFFFF if cin else 0) ^ Bs[j][i]
        carry[i] ^= bin(bal).count("1") & 1
    alt = 0
    for hyp in (0, 1):
        par = 0
        for j in range(nl):
            Xh = list(X[j])
            if hyp:
                Xh[2 * K] ^= 0xFFFFFFFF
            par ^= (pref(plane_e(2 * K + 1, Bs[j], Xh)) >> 31) & 1
        if hyp:
            alt ^= par
        else:
            carry[2 * K + 1] ^= par
    return carry, alt


def segmented_dual(data, h0, seglen):
    """Four dual passes + resolve (lzk_fnv_dual_pass_kernel /
    lzk_fnv_resolve_kernel), then the final pass + combine."""
    assert seglen % 1024 == 0
    segs = [data[k:k + seglen] for k in range(0, len(data), seglen)] or [b""]
    l0 = h0 & 0xFF
    par = [0] * len(segs)
    alt = [0] * len(segs)
    for K in range(4):
        for k, s in enumerate(segs[:-1]):
            lin = l0
            for q in par[:k]:
                lin ^= q
            cin = lin & ((1 << (2 * K)) - 1)
            carry = [(cin >> i) & 1 for i in range(8)]
            a = 0
            for c in range(0, len(s), 1024):
                carry, da = dual_chunk(s[c:c + 1024], carry, K)
                a ^= da
            par[k] |= (carry[2 * K] << (2 * K)) | (carry[2 * K + 1] << (2 * K + 1))
            alt[k] |= a << (2 * K + 1)
        bit = (l0 >> (2 * K)) & 1  # resolve: pick the hypothesis per segment
        for k in range(len(segs) - 1):
            if bit:
                par[k] = (par[k] & ~(1 << (2 * K + 1))) | (alt[k] & (1 << (2 * K + 1)))
            bit ^= (par[k] >> (2 * K)) & 1
    h = h0
    for k, s in enumerate(segs):
        lin = l0
        for q in par[:k]:
            lin ^= q
        assert lin == h & 0xFF, (k, lin, h & 0xFF)
        acc = fnv(s, lin)
        h = (pow(P, len(s), 1 << 64) * h + acc - pow(P, len(s), 1 << 64) * lin) & M64
    return h


if __name__ == "__main__":
    rng = random.Random(11)
    for n, sl in ((5 * 1024 + 77, 1024), (8 * 1024, 2048), (3 * 1024, 1024)):
        for trial in range(3):
            d = bytes(rng.getrandbits(8) for _ in range(n))
            h0 = rng.getrandbits(64)
            assert segmented_dual(d, h0, sl) == fnv(d, h0), (n, sl, trial)
    print("segmented dual ok")
