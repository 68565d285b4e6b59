"""TEST INFRASTRUCTURE ONLY: Python reference of the crypto members (C3/C4 workloads).

Each function restates the published algorithm the paper's crypto kernels implement
(ccminer SHA256d / Blake256 / Blake2B, ethminer Ethash) and is pinned on
standard test vectors in tests/test_crypto_oracle.py:
  * SHA-256d: hashlib (Bitcoin genesis block header -> 000000000019d6...)
  * BLAKE-256 (14 rounds): restated from the SHA-3 submission; pinned on its 1-byte and
    72-byte vectors
  * BLAKE2b-512: hashlib.blake2b
  * Keccak-256/512 (original 0x01 padding): restated; pinned on Keccak-256("") and
    Keccak-512("")
  * the Ethash-style hashimoto loop of the ethash member (synthetic DAG, ethminer's modulo walk:
    page = fnv(i ^ s[0], mix[i % 32]) mod n_pages, Ethash spec `hashimoto`; Keccak pinned)

Workload conventions (shared with paper_2007_01277_b200/kernels/gen_crypto.py): a header is
20 32-bit words; the nonce of thread-iteration n is nonce0 + n (32-bit wrap).
"""
import hashlib
import struct

import numpy as np

M32 = 0xFFFFFFFF


def rotr(x, n):
    return ((x >> n) | (x << (32 - n))) & M32


def bswap(x):
    return struct.unpack("<I", struct.pack(">I", x & M32))[0]


# ---- SHA-256d (Bitcoin) ---------------------------------------------------------------

def sha256d_header(words, nonce):
    """words: 20 header words (big-endian encoded); word 19 carries the nonce little-endian
    (Bitcoin byte order), i.e. word19 = bswap(nonce). Returns the 8 big-endian digest words."""
    w = [x & M32 for x in words]
    w[19] = bswap(nonce)
    data = b"".join(struct.pack(">I", x) for x in w)
    d = hashlib.sha256(hashlib.sha256(data).digest()).digest()
    return list(struct.unpack(">8I", d))


# ---- BLAKE-256 (14 rounds) ---------------------------------------------------------------

B256_IV = [0x6A09E667, 0xBB67AE85, 0x3C6EF372, 0xA54FF53A, 0x510E527F, 0x9B05688C, 0x1F83D9AB, 0x5BE0CD19]
B256_C = [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0, 0x082EFA98, 0xEC4E6C89,
          0x452821E6, 0x38D01377, 0xBE5466CF, 0x34E90C6C, 0xC0AC29B7, 0xC97C50DD, 0x3F84D5B5, 0xB5470917]
SIGMA = [
    [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15],
    [14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3],
    [11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4],
    [7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8],
    [9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13],
    [2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9],
    [12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11],
    [13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10],
    [6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5],
    [10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0],
]
G_IDX = [(0, 4, 8, 12), (1, 5, 9, 13), (2, 6, 10, 14), (3, 7, 11, 15),
         (0, 5, 10, 15), (1, 6, 11, 12), (2, 7, 8, 13), (3, 4, 9, 14)]


def blake256_compress(h, m, t):
    v = list(h) + B256_C[:4] + [t & M32 ^ B256_C[4], t & M32 ^ B256_C[5], (t >> 32) ^ B256_C[6],
                                (t >> 32) ^ B256_C[7]]
    for r in range(14):
        s = SIGMA[r % 10]
        for i, (a, b, c, d) in enumerate(G_IDX):
            x, y = s[2 * i], s[2 * i + 1]
            v[a] = (v[a] + v[b] + (m[x] ^ B256_C[y])) & M32
            v[d] = rotr(v[d] ^ v[a], 16)
            v[c] = (v[c] + v[d]) & M32
            v[b] = rotr(v[b] ^ v[c], 12)
            v[a] = (v[a] + v[b] + (m[y] ^ B256_C[x])) & M32
            v[d] = rotr(v[d] ^ v[a], 8)
            v[c] = (v[c] + v[d]) & M32
            v[b] = rotr(v[b] ^ v[c], 7)
    return [h[i] ^ v[i] ^ v[i + 8] for i in range(8)]


def blake256(msg: bytes) -> bytes:
    """BLAKE-256 (salt 0) of an arbitrary message."""
    nbits = len(msg) * 8
    padded = msg + b"\x80"
    while len(padded) % 64 != 56:
        padded += b"\x00"
    padded = padded[:-1] + bytes([padded[-1] | 0x01])  # the '1' bit before the length
    padded += struct.pack(">Q", nbits)
    h = list(B256_IV)
    nblocks = len(padded) // 64
    for i in range(nblocks):
        m = list(struct.unpack(">16I", padded[64 * i:64 * i + 64]))
        # counter = message bits processed up to and including this block; a block holding
        # only padding gets counter 0
        done = min(nbits, 512 * (i + 1))
        t = 0 if done <= 512 * i else done
        h = blake256_compress(h, m, t)
    return b"".join(struct.pack(">I", x) for x in h)


def blake256_header(words, nonce):
    """Header bytes = big-endian words; word 19 = nonce (big-endian). 8 digest words."""
    w = [x & M32 for x in words]
    w[19] = nonce & M32
    return list(struct.unpack(">8I", blake256(b"".join(struct.pack(">I", x) for x in w))))


# ---- BLAKE2b-512 -----------------------------------------------------------------------

def blake2b_header(words, nonce):
    """Header bytes = little-endian words; word 19 = nonce. Returns the 16 little-endian
    32-bit words of the 64-byte digest."""
    w = [x & M32 for x in words]
    w[19] = nonce & M32
    d = hashlib.blake2b(b"".join(struct.pack("<I", x) for x in w), digest_size=64).digest()
    return list(struct.unpack("<16I", d))


# ---- Keccak (original padding) and the ethash member -------------------------------------

RC = [0x0000000000000001, 0x0000000000008082, 0x800000000000808A, 0x8000000080008000, 0x000000000000808B,
      0x0000000080000001, 0x8000000080008081, 0x8000000000008009, 0x000000000000008A, 0x0000000000000088,
      0x0000000080008009, 0x000000008000000A, 0x000000008000808B, 0x800000000000008B, 0x8000000000008089,
      0x8000000000008003, 0x8000000000008002, 0x8000000000000080, 0x000000000000800A, 0x800000008000000A,
      0x8000000080008081, 0x8000000000008080, 0x0000000080000001, 0x8000000080008008]
ROT = [[0, 36, 3, 41, 18], [1, 44, 10, 45, 2], [62, 6, 43, 15, 61], [28, 55, 25, 21, 56], [27, 20, 39, 8, 14]]
M64 = (1 << 64) - 1


def keccak_f(A):
    """A[x][y], 64-bit lanes."""
    for rnd in range(24):
        C = [A[x][0] ^ A[x][1] ^ A[x][2] ^ A[x][3] ^ A[x][4] for x in range(5)]
        D = [C[(x - 1) % 5] ^ (((C[(x + 1) % 5] << 1) | (C[(x + 1) % 5] >> 63)) & M64) for x in range(5)]
        A = [[A[x][y] ^ D[x] for y in range(5)] for x in range(5)]
        B = [[0] * 5 for _ in range(5)]
        for x in range(5):
            for y in range(5):
                r = ROT[x][y]
                B[y][(2 * x + 3 * y) % 5] = ((A[x][y] << r) | (A[x][y] >> (64 - r))) & M64 if r else A[x][y]
        A = [[B[x][y] ^ ((~B[(x + 1) % 5][y]) & B[(x + 2) % 5][y]) for y in range(5)] for x in range(5)]
        A[0][0] ^= RC[rnd]
    return A


def keccak(data: bytes, rate: int, out_len: int) -> bytes:
    p = bytearray(data) + b"\x01"
    while len(p) % rate:
        p += b"\x00"
    p[-1] |= 0x80
    A = [[0] * 5 for _ in range(5)]
    for off in range(0, len(p), rate):
        blk = p[off:off + rate]
        for i in range(rate // 8):
            x, y = i % 5, i // 5
            A[x][y] ^= struct.unpack("<Q", blk[8 * i:8 * i + 8])[0]
        A = keccak_f(A)
    out = b"".join(struct.pack("<Q", A[i % 5][i // 5]) for i in range(25))
    return out[:out_len]


def keccak256(data):
    return keccak(data, 136, 32)


def keccak512(data):
    return keccak(data, 72, 64)


FNV_PRIME = 0x01000193


def fnv(a, b):
    return ((a * FNV_PRIME) ^ b) & M32


def ethash_hashimoto(header_words, nonce, dag, n_pages):
    """The ethash member: seed = Keccak-512(header_hash || nonce_le64); a 128-byte mix
    (32 words) initialised from the seed, 64 rounds of fnv-mixing with the DAG page
    p = fnv(i ^ seed[0], mix[i % 32]) mod n_pages (the Ethash spec's `hashimoto` walk over
    n_pages 128-byte pages, any count; the fnv word unsigned), 8-word
    compression, result = Keccak-256(seed || cmix). Returns (cmix[8], result words[8]),
    32-bit little-endian words. dag: numpy uint32 array of n_pages * 32 words."""
    hh = b"".join(struct.pack("<I", x & M32) for x in header_words[:8])
    seed = keccak512(hh + struct.pack("<Q", nonce & M32))
    s = list(struct.unpack("<16I", seed))
    mix = [s[i % 16] for i in range(32)]
    for i in range(64):
        p = fnv(i ^ s[0], mix[i % 32]) % n_pages
        page = dag[p * 32:(p + 1) * 32]
        mix = [fnv(mix[j], int(page[j])) for j in range(32)]
    cmix = [fnv(fnv(fnv(mix[4 * k], mix[4 * k + 1]), mix[4 * k + 2]), mix[4 * k + 3]) for k in range(8)]
    res = keccak256(seed + b"".join(struct.pack("<I", x) for x in cmix))
    return cmix, list(struct.unpack("<8I", res))


# ---- the kernels' outputs for a nonce range ------------------------------------------------

def search_outputs(kind, header_words, nonce0, count, target, grid, nthreads, dag=None, n_pages=0):
    """What a crypto member writes: cnt = #nonces with digest word < target (unsigned),
    chk = wrapping sum of digest word 0, bmin[b] = smallest hit nonce handled by block b
    (grid-stride assignment n -> block (n // nthreads) % grid), 0x7fffffff if none."""
    cnt, chk = 0, 0
    bmin = [0x7FFFFFFF] * grid
    for n in range(count):
        nonce = (nonce0 + n) & M32
        if kind == "sha256d":
            d = sha256d_header(header_words, nonce)
            word, crit = d[0], d[7]
        elif kind == "blake256":
            d = blake256_header(header_words, nonce)
            word, crit = d[0], d[0]
        elif kind == "blake2b":
            d = blake2b_header(header_words, nonce)
            word, crit = d[0], d[0]
        else:
            _, d = ethash_hashimoto(header_words, nonce, dag, n_pages)
            word, crit = d[0], d[0]
        chk = (chk + word) & M32
        if crit < target:
            cnt += 1
            b = (n // nthreads) % grid
            signed = nonce - (1 << 32) if nonce & 0x80000000 else nonce
            bmin[b] = min(bmin[b], signed)
    to_i32 = lambda x: x - (1 << 32) if x & 0x80000000 else x  # noqa: E731
    return {"cnt": cnt, "chk": to_i32(chk), "bmin": bmin}


def dag_words(seed, lo, hi, start, count):
    """Elements [start, start + count) of `array ... seed S range LO HI` (memimage.cpp:39-50)."""
    idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + idx * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    span = np.uint64(hi - lo + 1)
    return ((z % span).astype(np.int64) + lo).astype(np.int64) & 0xFFFFFFFF


class LazyDag:
    """Page-addressable view of the seeded synthetic DAG without materialising it."""

    def __init__(self, seed, npages):
        self.seed, self.npages = seed, npages

    def __getitem__(self, sl):
        return dag_words(self.seed, -2147483648, 2147483647, sl.start, sl.stop - sl.start)
