"""Generator of the crypto member kernels (MK+), the C3/C4 workloads of SURVEY §8d.

The paper's crypto kernels (ccminer SHA256d, Blake256, Blake2B and
ethminer's Ethash) have straight-line, fully unrolled rounds. Every member here is tunable (any
warp-multiple block size: nonces are strided by blockDim, the per-block minimum is indexed by the
block), so the partition search sizes both intervals of a fused pair — a 128-thread BLAKE-256
interval next to a 640-thread Ethash one beats the paper's fixed 512 + 512
(profiles/r02_probe_crypto_tunable.jsonl). Mini-Kernel
has no local arrays, so rounds are generated here as straight-line MK+ with statically
renamed state registers (no register moves), hex constants, 32-bit rotates (funnel shifts on
sm_100a) and 64-bit arithmetic in 32-bit halves (carry via `ltu`, rotates via `fshr`/`fshl`).
Header words are scalar kernel parameters: they live in the constant bank, and with JIT
specialization the nonce-independent first block (the midstate) folds at compile time.

Common contract of every kernel (prefix P):
  nonce of iteration n = P_nonce0 + n (32-bit wrap), n in [0, P_count), grid-stride;
  P_cnt[0]  += number of nonces whose criterion word is below P_target (unsigned);
  P_chk[0]  += digest word 0 (wrapping sum over all nonces);
  P_bmin[b] = smallest hit nonce of block b (0x7fffffff if none).
The Python restatement in oracle/crypto_ref.py (pinned on standard test vectors) computes the
same three outputs.

Run `python -m paper_2007_01277_b200.kernels.gen_crypto` to regenerate kernels/b200/*.mk.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))

SHA_K = [0x428A2F98, 0x71374491, 0xB5C0FBCF, 0xE9B5DBA5, 0x3956C25B, 0x59F111F1, 0x923F82A4, 0xAB1C5ED5,
         0xD807AA98, 0x12835B01, 0x243185BE, 0x550C7DC3, 0x72BE5D74, 0x80DEB1FE, 0x9BDC06A7, 0xC19BF174,
         0xE49B69C1, 0xEFBE4786, 0x0FC19DC6, 0x240CA1CC, 0x2DE92C6F, 0x4A7484AA, 0x5CB0A9DC, 0x76F988DA,
         0x983E5152, 0xA831C66D, 0xB00327C8, 0xBF597FC7, 0xC6E00BF3, 0xD5A79147, 0x06CA6351, 0x14292967,
         0x27B70A85, 0x2E1B2138, 0x4D2C6DFC, 0x53380D13, 0x650A7354, 0x766A0ABB, 0x81C2C92E, 0x92722C85,
         0xA2BFE8A1, 0xA81A664B, 0xC24B8B70, 0xC76C51A3, 0xD192E819, 0xD6990624, 0xF40E3585, 0x106AA070,
         0x19A4C116, 0x1E376C08, 0x2748774C, 0x34B0BCB5, 0x391C0CB3, 0x4ED8AA4A, 0x5B9CCA4F, 0x682E6FF3,
         0x748F82EE, 0x78A5636F, 0x84C87814, 0x8CC70208, 0x90BEFFFA, 0xA4506CEB, 0xBEF9A3F7, 0xC67178F2]
IV256 = [0x6A09E667, 0xBB67AE85, 0x3C6EF372, 0xA54FF53A, 0x510E527F, 0x9B05688C, 0x1F83D9AB, 0x5BE0CD19]
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
IV512 = [0x6A09E667F3BCC908, 0xBB67AE8584CAA73B, 0x3C6EF372FE94F82B, 0xA54FF53A5F1D36F1,
         0x510E527FADE682D1, 0x9B05688C2B3E6C1F, 0x1F83D9ABFB41BD6B, 0x5BE0CD19137E2179]
RC = [0x0000000000000001, 0x0000000000008082, 0x800000000000808A, 0x8000000080008000, 0x000000000000808B,
      0x0000000080000001, 0x8000000080008081, 0x8000000000008009, 0x000000000000008A, 0x0000000000000088,
      0x0000000080008009, 0x000000008000000A, 0x000000008000808B, 0x800000000000008B, 0x8000000000008089,
      0x8000000000008003, 0x8000000000008002, 0x8000000000000080, 0x000000000000800A, 0x800000008000000A,
      0x8000000080008081, 0x8000000000008080, 0x0000000080000001, 0x8000000080008008]
HPP = int(os.environ.get("HF_ETHASH_HPP", "8"))  # Ethash: nonces of an 8-lane group whose DAG walks are in flight together per lane
# Ethash DAG reads: "ldg" = 128-bit register loads (vload); "async" = 16-byte cp.async copies into a
# per-thread shared-memory ring (MK+ async_copy / async_wait), so no register holds a page in flight
ETHASH_LOAD = os.environ.get("HF_ETHASH_LOAD", "ldg")
ETHASH_TMAX = 512  # async form: the shared ring is sized for intervals of up to 512 threads
# "lean" form: cp.async DAG ring + the Keccak-512 seed parked in shared memory across the DAG walk,
# so the walk holds only the mixes (32 registers) and the page indices: twice the resident warps
# (pages in flight) of the register form. Its shared arrays are sized for intervals of up to
# ETHASH_LEAN_TMAX threads (8 x 16 B ring + 64 B seed per thread).
# The lean form is the default member (every Ethash pair fuses 5-13 % faster with it, r02 probe);
# the register form (ethash_reg.mk) is kept because it is ~5 % faster ALONE: the bench's unfused
# baselines run whichever form is faster, so a fused win is never a win over a slowed member.
ETHASH_FORM = os.environ.get("HF_ETHASH_FORM", "lean")
ETHASH_LEAN_TMAX = int(os.environ.get("HF_ETHASH_TMAX", "1024"))
# Keccak-f as 24 straight-line rounds with immediate round constants (HF_KECCAK_UNROLL=1) instead
# of a rolled round loop reading the constants from eh_rc (probe: register pressure / spills of the
# lean Ethash member at 64 registers)
KECCAK_UNROLL = os.environ.get("HF_KECCAK_UNROLL", "") == "1"
ROT = [[0, 36, 3, 41, 18], [1, 44, 10, 45, 2], [62, 6, 43, 15, 61], [28, 55, 25, 21, 56], [27, 20, 39, 8, 14]]


def hx(v):
    return f"0x{v & 0xFFFFFFFF:08x}"


class Src:
    def __init__(self):
        self.lines = []
        self.ind = 1

    def __call__(self, s=""):
        self.lines.append("  " * self.ind + s if s else "")

    def text(self):
        return "\n".join(self.lines) + "\n"


def decls(src, names, ty="int"):
    for i in range(0, len(names), 12):
        src(" ".join(f"{ty} {n};" for n in names[i:i + 12]))


def header(src, p, kind, doc, params, dims, shared=True, fixed=False):
    src.lines.append(doc.rstrip())
    src.lines.append("//@ grid=296")
    src.lines.append(f"kernel {kind}({params}) dims ({dims}, 1, 1){' fixed' if fixed else ''} {{")
    if shared:
        src(f"shared int {p}_smin[32];")


def tail(src, p):
    """Per-block min of the hit nonces: 5-step shuffle tree, one smem stage, warp 0 folds."""
    src(f"best = min(best, warp_shfl_xor(best, 16));")
    src(f"best = min(best, warp_shfl_xor(best, 8));")
    src(f"best = min(best, warp_shfl_xor(best, 4));")
    src(f"best = min(best, warp_shfl_xor(best, 2));")
    src(f"best = min(best, warp_shfl_xor(best, 1));")
    src(f"if (tid % 32 == 0) {{")
    src(f"  {p}_smin[tid / 32] = best;")
    src("}")
    src("syncthreads();")
    src("if (tid < 32) {")
    src(f"  best = 2147483647;")
    src(f"  if (tid < nthr / 32) {{")
    src(f"    best = {p}_smin[tid];")
    src("  }")
    for m in (16, 8, 4, 2, 1):
        src(f"  best = min(best, warp_shfl_xor(best, {m}));")
    src("  if (tid == 0) {")
    src(f"    {p}_bmin[blockIdx.x] = best;")
    src("  }")
    src("}")
    src.ind = 0
    src("}")


def loop_head(src, p):
    src(f"int tid = threadIdx.x;")
    src(f"int nthr = blockDim.x;")
    src(f"int best = 2147483647;")
    src(f"int cnt = 0;")
    src(f"int chk = 0;")


def loop_open(src, p):
    src(f"for (int n = blockIdx.x * nthr + tid; n < {p}_count; n = n + gridDim.x * nthr) {{")
    src.ind += 1
    src(f"int nonce = {p}_nonce0 + n;")


def loop_close(src, p, word, crit):
    src(f"chk = chk + {word};")
    src(f"if (ltu({crit}, {p}_target)) {{")
    src("  cnt = cnt + 1;")
    src("  best = min(best, nonce);")
    src("}")
    src.ind -= 1
    src("}")
    src(f"atomic_add({p}_chk[0], chk);")
    src(f"if (cnt > 0) {{")
    src(f"  atomic_add({p}_cnt[0], cnt);")
    src("}")


# ---------------------------------------------------------------------------------------
# SHA-256d
# ---------------------------------------------------------------------------------------

# SHA-256 pipe balance (HF_SHA_PIPES): "alu" = every rotate/shift a funnel shift (SHF) and every
# add an IADD3, all on the ALU pipe, which SHA-256d saturates (98 % busy, FMA pipe 5 %);
# "fma" = two of the three rotates of each Sigma/sigma and the sigma shifts as multiplies by a
# power of two held in a register (x << k = x * 2^k: IMAD; x >> (32 - k) = mulhi_u(x, 2^k):
# IMAD.HI; the halves of a rotate have disjoint bits, so they join the Sigma's XOR directly),
# which moves about a third of the round's work to the idle FMA pipe. The powers come from the
# sh_pw array (a register the compiler cannot fold into a shift). Measured on B200: ptxas turns each
# rotate half-pair into one IMAD.WIDE.U32, which is far slower than the SHF it replaces (SHA-256d
# alone 2,846 vs 2,138 us, every fused pair 16-20 % slower; profiles/r02_probe_sha_pipes.jsonl), so
# the member keeps "alu".
SHA_PIPES = os.environ.get("HF_SHA_PIPES", "alu")
SHA_POW = {26: "pw26", 21: "pw21", 30: "pw30", 19: "pw19", 25: "pw25", 14: "pw14", 15: "pw15", 13: "pw13",
           29: "pw29", 22: "pw22"}


def _rot_fma(x, n):
    """rotr(x, n) as the XOR of its two disjoint halves, both on the FMA pipe."""
    k = SHA_POW[32 - n]
    return f"({x} * {k}) ^ mulhi_u({x}, {k})"


def _shr_fma(x, n):
    return f"mulhi_u({x}, {SHA_POW[32 - n]})"


# SHA-256 adds (HF_SHA_ADDS): "fma" writes every add of the round and the schedule as MK+
# fma_add (IMAD a, one, b on the FMA pipe), leaving the ALU pipe the rotates and LOP3s only.
SHA_ADDS = os.environ.get("HF_SHA_ADDS", "")


def _sum(terms, fma):
    """terms[0] + terms[1] + ...; with fma a left-to-right fma_add chain."""
    if not fma:
        return " + ".join(terms)
    acc = terms[0]
    for t in terms[1:]:
        acc = f"fma_add({acc}, {t})"
    return acc


def sha_rounds(src, roles, w, first_w=None):
    """64 rounds; roles = list of 8 variable names (a..h); w = 16 schedule variable names.
    Returns the final roles."""
    R = list(roles)
    fma = SHA_PIPES == "fma"
    fa = SHA_ADDS == "fma"
    for i in range(64):
        if i >= 16:
            x, x2, x7, x15 = w[i % 16], w[(i - 2) % 16], w[(i - 7) % 16], w[(i - 15) % 16]
            if fma:
                src(f"{x} = ({_rot_fma(x2, 17)} ^ {_rot_fma(x2, 19)} ^ {_shr_fma(x2, 10)}) + {x7} + "
                    f"({_rot_fma(x15, 7)} ^ {_rot_fma(x15, 18)} ^ {_shr_fma(x15, 3)}) + {x};")
            else:
                src(f"{x} = " + _sum([f"(rotr({x2}, 17) ^ rotr({x2}, 19) ^ shr_u({x2}, 10))", x7,
                                      f"(rotr({x15}, 7) ^ rotr({x15}, 18) ^ shr_u({x15}, 3))", x], fa) + ";")
        a, b, c, d, e, f, g, h = R
        if fma:
            s1 = f"({_rot_fma(e, 6)} ^ {_rot_fma(e, 11)} ^ rotr({e}, 25))"
            s0 = f"({_rot_fma(a, 2)} ^ {_rot_fma(a, 13)} ^ rotr({a}, 22))"
        else:
            s1 = f"(rotr({e}, 6) ^ rotr({e}, 11) ^ rotr({e}, 25))"
            s0 = f"(rotr({a}, 2) ^ rotr({a}, 13) ^ rotr({a}, 22))"
        src("t1 = " + _sum([h, s1, f"({g} ^ ({e} & ({f} ^ {g})))", hx(SHA_K[i]), w[i % 16]], fa) + ";")
        src("t2 = " + _sum([s0, f"(({a} & {b}) | ({c} & ({a} | {b})))"], fa) + ";")
        src(f"{d} = " + _sum([d, "t1"], fa) + ";")
        src(f"{h} = " + _sum(["t1", "t2"], fa) + ";")
        R = [h, a, b, c, d, e, f, g]
    return R


def gen_sha256d():
    p = "sh"
    s = Src()
    hp = ", ".join(f"int {p}_h{i}" for i in range(19))
    header(s, p, "sha256d", """// SHA-256d nonce search (Bitcoin header hashing; ccminer sha256d analogue, PAPER.md:876).
// Generated by kernels/gen_crypto.py. Header = 20 big-endian words (scalar params h0..h18,
// word 19 = bswap(nonce)); digest = SHA256(SHA256(header)); criterion word = digest[7].
// The nonce-independent first block (the midstate) is compressed once per thread.""",
           f"int {p}_cnt[], int {p}_chk[], int {p}_bmin[], {hp}, int {p}_nonce0, int {p}_count, int {p}_target"
           + (f", int {p}_pw[]" if SHA_PIPES == "fma" else ""), 512)
    st = [f"s{c}" for c in "abcdefgh"]
    w = [f"w{i}" for i in range(16)]
    mid = [f"m{i}" for i in range(8)]
    dig = [f"d{i}" for i in range(8)]
    decls(s, st + w + mid + dig + ["t1", "t2"])
    loop_head(s, p)
    if SHA_PIPES == "fma":
        for k, v in sorted(SHA_POW.items()):
            s(f"int {v} = {p}_pw[{k}];")
    for i in range(8):
        s(f"{st[i]} = {hx(IV256[i])};")
    for i in range(16):
        s(f"{w[i]} = {p}_h{i};")
    R = sha_rounds(s, st, w)
    for i in range(8):
        s(f"{mid[i]} = {hx(IV256[i])} + {R[i]};")
    loop_open(s, p)
    # block 2: header words 16..18, bswap(nonce), padding, length 640
    s(f"w0 = {p}_h16;")
    s(f"w1 = {p}_h17;")
    s(f"w2 = {p}_h18;")
    s("w3 = (nonce << 24) | ((nonce << 8) & 0x00ff0000) | (shr_u(nonce, 8) & 0x0000ff00) | shr_u(nonce, 24);")
    s("w4 = 0x80000000;")
    for i in range(5, 15):
        s(f"w{i} = 0;")
    s("w15 = 640;")
    for i in range(8):
        s(f"{st[i]} = {mid[i]};")
    R = sha_rounds(s, st, w)
    for i in range(8):
        s(f"{dig[i]} = {mid[i]} + {R[i]};")
    # second SHA-256 over the 32-byte digest
    for i in range(8):
        s(f"w{i} = {dig[i]};")
    s("w8 = 0x80000000;")
    for i in range(9, 15):
        s(f"w{i} = 0;")
    s("w15 = 256;")
    for i in range(8):
        s(f"{st[i]} = {hx(IV256[i])};")
    R = sha_rounds(s, st, w)
    for i in range(8):
        s(f"{dig[i]} = {hx(IV256[i])} + {R[i]};")
    loop_close(s, p, "d0", "d7")
    tail(s, p)
    return s.text()


# ---------------------------------------------------------------------------------------
# BLAKE-256 (14 rounds)
# ---------------------------------------------------------------------------------------

# BLAKE-256 pipe balance (HF_B256_ADDS): the G function's adds are the only work of the round
# that can leave the ALU pipe (XORs and rotates are LOP3/SHF, ALU-only); each letter moves one
# add site onto the FMA pipe as MK+ fma_add (IMAD a, one, b): "a" = a = a + b + (m ^ c) (two
# IMADs), "c" = c = c + d (one IMAD). "" keeps every add an IADD3 on the ALU pipe.
B256_ADDS = os.environ.get("HF_B256_ADDS", "")


def _add(x, y, fma):
    return f"fma_add({x}, {y})" if fma else f"{x} + {y}"


def blake256_compress(src, h, m, t, v):
    """m: 16 expressions (variable names or hex literals); t: counter (python int)."""
    fa, fc = "a" in B256_ADDS, "c" in B256_ADDS
    for i in range(8):
        src(f"{v[i]} = {h[i]};")
    for i in range(4):
        src(f"{v[8 + i]} = {hx(B256_C[i])};")
    src(f"{v[12]} = {hx(t ^ B256_C[4])};")
    src(f"{v[13]} = {hx(t ^ B256_C[5])};")
    src(f"{v[14]} = {hx(B256_C[6])};")
    src(f"{v[15]} = {hx(B256_C[7])};")
    for r in range(14):
        sg = SIGMA[r % 10]
        for i, (a, b, c, d) in enumerate(G_IDX):
            x, y = sg[2 * i], sg[2 * i + 1]
            A, B, Cc, D = v[a], v[b], v[c], v[d]
            src(f"{A} = {_add(_add(A, B, fa), f'({m[x]} ^ {hx(B256_C[y])})', fa)};")
            src(f"{D} = rotr({D} ^ {A}, 16);")
            src(f"{Cc} = {_add(Cc, D, fc)};")
            src(f"{B} = rotr({B} ^ {Cc}, 12);")
            src(f"{A} = {_add(_add(A, B, fa), f'({m[y]} ^ {hx(B256_C[x])})', fa)};")
            src(f"{D} = rotr({D} ^ {A}, 8);")
            src(f"{Cc} = {_add(Cc, D, fc)};")
            src(f"{B} = rotr({B} ^ {Cc}, 7);")


def gen_blake256():
    p = "bl"
    s = Src()
    hp = ", ".join(f"int {p}_h{i}" for i in range(19))
    header(s, p, "blake256", """// BLAKE-256 (14 rounds) nonce search (ccminer blake256 analogue, PAPER.md:876).
// Generated by kernels/gen_crypto.py. Message = 80-byte header of big-endian words (scalar
// params h0..h18, word 19 = nonce); two compressions (t = 512, t = 640); the first is
// nonce-independent (midstate, once per thread). Criterion and checksum word = digest[0].""",
           f"int {p}_cnt[], int {p}_chk[], int {p}_bmin[], {hp}, int {p}_nonce0, int {p}_count, int {p}_target",
           512)
    v = [f"v{i}" for i in range(16)]
    mid = [f"m{i}" for i in range(8)]
    decls(s, v + mid + ["h0", "h1", "h2", "h3", "h4", "h5", "h6", "h7"])
    loop_head(s, p)
    blake256_compress(s, [hx(x) for x in IV256], [f"{p}_h{i}" for i in range(16)], 512, v)
    for i in range(8):
        s(f"{mid[i]} = {hx(IV256[i])} ^ {v[i]} ^ {v[i + 8]};")
    loop_open(s, p)
    msg = [f"{p}_h16", f"{p}_h17", f"{p}_h18", "nonce", hx(0x80000000)] + ["0"] * 8 + ["1", "0", "640"]
    blake256_compress(s, mid, msg, 640, v)
    for i in range(8):
        s(f"h{i} = {mid[i]} ^ {v[i]} ^ {v[i + 8]};")
    loop_close(s, p, "h0", "h0")
    tail(s, p)
    return s.text()


# ---------------------------------------------------------------------------------------
# BLAKE2b-512 (64-bit lanes as 32-bit halves)
# ---------------------------------------------------------------------------------------

class Lane:
    """A 64-bit value held in two 32-bit variables; swap() renames (rotr by 32 is free)."""

    def __init__(self, lo, hi):
        self.lo, self.hi = lo, hi


# How 64-bit adds carry (BLAKE2b): "ltu" = unsigned compare + select (ISETP + IMAD: the select
# runs on the FMA pipe), "addc" = MK+ addc (add.cc/addc: IADD3 + IADD3.X, fewer instructions but
# all on the ALU pipe), "mix" = alternate. See profiles/r01_probe_blake2b_carry.json.
ADD64 = os.environ.get("HF_ADD64", "ltu")
_add64_n = [0]


def _use_addc():
    _add64_n[0] += 1
    return ADD64 == "addc" or (ADD64 == "mix" and _add64_n[0] % 2 == 0)


def _add64(src, a, hi_b, lo_b):
    if _use_addc():
        src(f"{a.hi} = addc({a.hi}, {hi_b}, {a.lo}, {lo_b});")
        src(f"{a.lo} = {a.lo} + {lo_b};")
    else:
        src(f"t = {a.lo} + {lo_b};")
        src(f"{a.hi} = {a.hi} + {hi_b} + ltu(t, {a.lo});")
        src(f"{a.lo} = t;")


def add64(src, a, b):
    _add64(src, a, b.hi, b.lo)


def add64_m(src, a, m):
    """a += m where m = (lo_expr, hi_expr)."""
    lo, hi = m
    if lo == "0" and hi == "0":
        return
    _add64(src, a, hi, lo)


def xor64(src, a, b):
    src(f"{a.lo} = {a.lo} ^ {b.lo};")
    src(f"{a.hi} = {a.hi} ^ {b.hi};")


def rotr64(src, a, r):
    if r == 32:
        a.lo, a.hi = a.hi, a.lo
        return
    if r > 32:
        a.lo, a.hi = a.hi, a.lo
        r -= 32
    src(f"t = fshr({a.lo}, {a.hi}, {r});")
    src(f"{a.hi} = fshr({a.hi}, {a.lo}, {r});")
    src(f"{a.lo} = t;")


def gen_blake2b():
    p = "b2"
    s = Src()
    hp = ", ".join(f"int {p}_h{i}" for i in range(19))
    header(s, p, "blake2b", """// BLAKE2b-512 nonce search (ccminer blake2b analogue, PAPER.md:876).
// Generated by kernels/gen_crypto.py. Message = 80-byte header of little-endian words
// (scalar params h0..h18, word 19 = nonce): one compression with t = 80 and the final flag.
// 64-bit lanes live in 32-bit halves: adds carry through """ + ("ltu (compare + select)" if ADD64 == "ltu" else "addc (add.cc/addc)" if ADD64 == "addc" else "alternately ltu and addc") + """, rotates are funnel shifts
// (SHF on sm_100a) and rotations by 32 are free renames. Criterion/checksum word = the low
// 32 bits of digest lane 0.""",
           f"int {p}_cnt[], int {p}_chk[], int {p}_bmin[], {hp}, int {p}_nonce0, int {p}_count, int {p}_target",
           512)
    names = []
    for i in range(16):
        names += [f"v{i}l", f"v{i}h"]
    decls(s, names + ["t", "o0"])
    loop_head(s, p)
    loop_open(s, p)
    words = [f"{p}_h{i}" for i in range(19)] + ["nonce"]
    m = [(words[2 * k], words[2 * k + 1]) for k in range(10)] + [("0", "0")] * 6
    v = [Lane(f"v{i}l", f"v{i}h") for i in range(16)]
    h0 = list(IV512)
    h0[0] ^= 0x01010040
    for i in range(8):
        s(f"{v[i].lo} = {hx(h0[i])};")
        s(f"{v[i].hi} = {hx(h0[i] >> 32)};")
    for i in range(8):
        iv = IV512[i]
        if i == 4:
            iv ^= 80
        if i == 6:
            iv ^= 0xFFFFFFFFFFFFFFFF
        s(f"{v[8 + i].lo} = {hx(iv)};")
        s(f"{v[8 + i].hi} = {hx(iv >> 32)};")
    for r in range(12):
        sg = SIGMA[r % 10]
        for i, (a, b, c, d) in enumerate(G_IDX):
            A, B, Cc, D = v[a], v[b], v[c], v[d]
            add64(s, A, B)
            add64_m(s, A, m[sg[2 * i]])
            xor64(s, D, A)
            rotr64(s, D, 32)
            add64(s, Cc, D)
            xor64(s, B, Cc)
            rotr64(s, B, 24)
            add64(s, A, B)
            add64_m(s, A, m[sg[2 * i + 1]])
            xor64(s, D, A)
            rotr64(s, D, 16)
            add64(s, Cc, D)
            xor64(s, B, Cc)
            rotr64(s, B, 63)
    s(f"o0 = {hx(h0[0])} ^ {v[0].lo} ^ {v[8].lo};")
    loop_close(s, p, "o0", "o0")
    tail(s, p)
    return s.text()


# ---------------------------------------------------------------------------------------
# Ethash-style hashimoto: Keccak-512 seed, 64 DAG page mixes, Keccak-256 result
# ---------------------------------------------------------------------------------------

PI_CYCLE = [(1, 0), (0, 2), (2, 1), (1, 2), (2, 3), (3, 3), (3, 0), (0, 1), (1, 3), (3, 1), (1, 4), (4, 4),
            (4, 0), (0, 3), (3, 4), (4, 3), (3, 2), (2, 2), (2, 0), (0, 4), (4, 2), (2, 4), (4, 1), (1, 1)]


def rotl64_into(src, dst_lo, dst_hi, lo, hi, r):
    if r >= 32:
        lo, hi = hi, lo
        r -= 32
    if r == 0:
        src(f"{dst_lo} = {lo};")
        src(f"{dst_hi} = {hi};")
    else:
        src(f"{dst_lo} = fshl({hi}, {lo}, {r});")
        src(f"{dst_hi} = fshl({lo}, {hi}, {r});")


def keccak_f(src, A, rc_array):
    """A: dict (x, y) -> Lane (current variable names). Emits the 24-round permutation as a
    loop over one straight-line, low-register round: theta with 5 column parities, rho+pi in
    place along the 24-lane pi cycle (one carried lane), chi row by row (5 saved lanes); the
    round constants come from rc_array (48 words)."""
    C = [Lane(f"c{x}l", f"c{x}h") for x in range(5)]
    D = Lane("dl", "dh")
    if KECCAK_UNROLL:
        for r in range(24):
            _keccak_round(src, A, C, D, hx(RC[r]), hx(RC[r] >> 32))
        return
    src("for (int rnd = 0; rnd < 24; rnd = rnd + 1) {")
    src.ind += 1
    _keccak_round(src, A, C, D, f"{rc_array}[rnd * 2]", f"{rc_array}[rnd * 2 + 1]")
    src.ind -= 1
    src("}")


def _keccak_round(src, A, C, D, rc_lo, rc_hi):
    for x in range(5):
        for half in ("lo", "hi"):
            terms = " ^ ".join(getattr(A[(x, y)], half) for y in range(5))
            src(f"{getattr(C[x], half)} = {terms};")
    for x in range(5):
        c1, c4 = C[(x + 1) % 5], C[(x - 1) % 5]
        # D = C[x-1] ^ rotl64(C[x+1], 1)
        src(f"{D.lo} = {c4.lo} ^ fshl({c1.hi}, {c1.lo}, 1);")
        src(f"{D.hi} = {c4.hi} ^ fshl({c1.lo}, {c1.hi}, 1);")
        for y in range(5):
            src(f"{A[(x, y)].lo} = {A[(x, y)].lo} ^ {D.lo};")
            src(f"{A[(x, y)].hi} = {A[(x, y)].hi} ^ {D.hi};")
    # rho + pi in place: the lane at p moves to pi(p) = (y, 2x + 3y) rotated by ROT[p]
    src(f"tl = {A[PI_CYCLE[0]].lo};")
    src(f"th = {A[PI_CYCLE[0]].hi};")
    for i, pos in enumerate(PI_CYCLE):
        dst = PI_CYCLE[(i + 1) % 24]
        x, y = pos
        if i < 23:
            src(f"ul = {A[dst].lo};")
            src(f"uh = {A[dst].hi};")
        rotl64_into(src, A[dst].lo, A[dst].hi, "tl", "th", ROT[x][y])
        if i < 23:
            src("tl = ul;")
            src("th = uh;")
    # chi row by row, iota from the round-constant table
    for y in range(5):
        for x in range(5):
            src(f"{C[x].lo} = {A[(x, y)].lo};")
            src(f"{C[x].hi} = {A[(x, y)].hi};")
        for x in range(5):
            b1, b2 = C[(x + 1) % 5], C[(x + 2) % 5]
            src(f"{A[(x, y)].lo} = {C[x].lo} ^ (({b1.lo} ^ -1) & {b2.lo});")
            src(f"{A[(x, y)].hi} = {C[x].hi} ^ (({b1.hi} ^ -1) & {b2.hi});")
    if rc_lo != "0x00000000":
        src(f"{A[(0, 0)].lo} = {A[(0, 0)].lo} ^ {rc_lo};")
    if rc_hi != "0x00000000":
        src(f"{A[(0, 0)].hi} = {A[(0, 0)].hi} ^ {rc_hi};")


def absorb_words(src, A, words):
    """XOR 32-bit words (little-endian lane order) into the zero state: lane i = words[2i], [2i+1]."""
    for i in range(25):
        x, y = i % 5, i // 5
        lo = words[2 * i] if 2 * i < len(words) else "0"
        hi = words[2 * i + 1] if 2 * i + 1 < len(words) else "0"
        src(f"{A[(x, y)].lo} = {lo};")
        src(f"{A[(x, y)].hi} = {hi};")


def bcast8(src, var, lane_src, tmp="bt"):
    """Broadcast `var` from group lane `lane_src` (0..7, the same for the 8 lanes of a group) to
    the 8 lanes of each 8-lane group: MK+ warp_bcast, one shfl.idx on the B200 (its lowering for
    the interpreter is the 3-step xor butterfly this helper used to spell out)."""
    src(f"{var} = warp_bcast({var}, {lane_src}, 8);")


def gen_ethash():
    if ETHASH_FORM == "lean":
        return gen_ethash_lean()
    p = "eh"
    s = Src()
    hp = ", ".join(f"int {p}_h{i}" for i in range(8))
    header(s, p, "ethash", """// Ethash-style hashimoto nonce search (ethminer analogue, PAPER.md:876-879).
// Generated by kernels/gen_crypto.py. seed = Keccak-512(header_hash[8 words] || nonce as
// 64-bit LE); mix = seed repeated to 32 words; 64 rounds: page = fnv(i ^ seed[0],
// mix[i % 32]) % npages (ethminer's modulo walk; remu: the fnv word read as uint32),
// mix = fnv(mix, dag[page]) over the 128-byte page;
// cmix = 8-word fnv fold; result = Keccak-256(seed || cmix).
// B200 mechanics (ethminer's lane-cooperative layout): every thread computes the two Keccaks
// of its own nonce, but the DAG loop of the 8 nonces of an 8-lane group is shared: lane j
// holds words 4j..4j+3 of """ + str(HPP) + """ of the group's mixes at a time, the lane owning mix[i % 32]
// computes each page index and broadcasts it (warp_bcast: one shfl.idx), and each DAG page is
// read by the 8 lanes as one coalesced 128-byte segment (""" + str(HPP) + """ pages in flight per lane
// per round, 4 lines per warp load instead of 32; 8 in flight measured 7% faster than 4 on B200). Keccak-f[1600] lanes are 32-bit halves (funnel-shift rotates, chi as
// LOP3, rho+pi in place along the pi cycle, chi row by row: ~64 live registers), 24 rounds as
// a loop over one straight-line round (constants from P_rc[48]).
// Criterion/checksum word = result word 0 (little-endian). The DAG is a synthetic
// page array of npages 128-byte pages (a prime count, like the real DAG's; any count < 2^25 works) (SURVEY §8d: a seeded int32 array, >= 4 GiB for C3). Any warp-
// multiple block size works (tunable: the partition search sizes it against its partner).""",
           f"int {p}_cnt[], int {p}_chk[], int {p}_bmin[], int {p}_dag[], int {p}_rc[], {hp}, int {p}_npages, "
           f"int {p}_nonce0, int {p}_count, int {p}_target", 256, fixed=False)
    if ETHASH_LOAD == "async":
        s(f"shared int {p}_ring[{HPP * ETHASH_TMAX * 4}];")
    A = {(x, y): Lane(f"a{x}{y}l", f"a{x}{y}h") for x in range(5) for y in range(5)}
    names = []
    for x in range(5):
        for y in range(5):
            names += [f"a{x}{y}l", f"a{x}{y}h"]
    for x in range(5):
        names += [f"c{x}l", f"c{x}h"]
    names += ["dl", "dh"] + [f"sd{i}" for i in range(16)] + [f"cm{i}" for i in range(8)]
    names += [f"x{h}_{k}" for h in range(HPP) for k in range(4)] + [f"z{h}" for h in range(HPP)]
    names += [f"pg{h}" for h in range(HPP)] + ["q0", "q1", "q2", "q3", "bt", "bw", "cw", "r0", "lj", "valid", "nonce"]
    names += ["tl", "th", "ul", "uh"]
    decls(s, names)
    s("int tid = threadIdx.x;")
    s("int nthr = blockDim.x;")
    s("int best = 2147483647;")
    s("int cnt = 0;")
    s("int chk = 0;")
    s("int lane = tid % 32;")
    s("lj = lane % 8;")
    s(f"for (int n0 = blockIdx.x * nthr + (tid / 32) * 32; n0 < {p}_count; n0 = n0 + gridDim.x * nthr) {{")
    s.ind += 1
    s("valid = n0 + lane < " + f"{p}_count;")
    s(f"nonce = {p}_nonce0 + n0 + lane;")
    # Keccak-512: rate 72 bytes = 9 lanes; input 40 bytes = 10 words, pad 0x01 at byte 40,
    # 0x80 at byte 71 (word 17, top byte)
    words = [f"{p}_h{i}" for i in range(8)] + ["nonce", "0", "0x00000001"] + ["0"] * 6 + ["0x80000000"]
    absorb_words(s, A, words)
    keccak_f(s, A, f"{p}_rc")
    for i in range(8):
        ln = A[(i % 5, i // 5)]
        s(f"sd{2 * i} = {ln.lo};")
        s(f"sd{2 * i + 1} = {ln.hi};")
    # The group's 8 nonces are processed HPP at a time: lane j keeps words 4j..4j+3 of the
    # mixes of nonces hg .. hg+HPP-1 (= seed words 4(j % 4) .. of those nonces).
    s(f"for (int hg = 0; hg < 8; hg = hg + {HPP}) {{")
    s.ind += 1
    for h in range(HPP):
        for w in range(16):
            s(f"bw = sd{w};")
            bcast8(s, "bw", f"(hg + {h})")
            if w == 0:
                s(f"z{h} = bw;")
            s(f"if (lj % 4 == {w // 4}) {{")
            s(f"  x{h}_{w % 4} = bw;")
            s("}")
    s("for (int it = 0; it < 64; it = it + 4) {")
    s.ind += 1
    s("int owner = (it % 32) / 4;")
    for k in range(4):
        for h in range(HPP):
            s(f"pg{h} = ((it + {k}) ^ z{h}) * 16777619 ^ x{h}_{k};")
            bcast8(s, f"pg{h}", "owner")
            s(f"pg{h} = remu(pg{h}, {p}_npages) * 8 + lj;")
        if ETHASH_LOAD == "async":
            for h in range(HPP):
                s(f"async_copy({p}_ring, {h * ETHASH_TMAX} + tid, {p}_dag, pg{h});")
            s("async_wait();")
        for h in range(HPP):
            if ETHASH_LOAD == "async":
                s(f"vload({p}_ring, {h * ETHASH_TMAX} + tid, q0, q1, q2, q3);")
            else:
                s(f"vload({p}_dag, pg{h}, q0, q1, q2, q3);")
            for j in range(4):
                s(f"x{h}_{j} = x{h}_{j} * 16777619 ^ q{j};")
    s.ind -= 1
    s("}")
    # cmix word j of nonce hg+h sits in lane j; transpose so each lane keeps its own nonce's
    for h in range(HPP):
        s(f"cw = ((x{h}_0 * 16777619 ^ x{h}_1) * 16777619 ^ x{h}_2) * 16777619 ^ x{h}_3;")
        for k in range(8):
            s("bw = cw;")
            bcast8(s, "bw", k)
            s(f"if (lj == hg + {h}) {{")
            s(f"  cm{k} = bw;")
            s("}")
    s.ind -= 1
    s("}")
    # Keccak-256: rate 136 bytes = 17 lanes; input 96 bytes = 24 words, pad 0x01 at byte 96,
    # 0x80 at byte 135 (word 33, top byte)
    words = [f"sd{i}" for i in range(16)] + [f"cm{i}" for i in range(8)] + ["0x00000001"] + ["0"] * 8 + ["0x80000000"]
    absorb_words(s, A, words)
    keccak_f(s, A, f"{p}_rc")
    s(f"r0 = {A[(0, 0)].lo};")
    s("if (valid) {")
    s("  chk = chk + r0;")
    s(f"  if (ltu(r0, {p}_target)) {{")
    s("    cnt = cnt + 1;")
    s("    best = min(best, nonce);")
    s("  }")
    s("}")
    s.ind -= 1
    s("}")
    s(f"atomic_add({p}_chk[0], chk);")
    s("if (cnt > 0) {")
    s(f"  atomic_add({p}_cnt[0], cnt);")
    s("}")
    tail(s, p)
    return s.text()


def gen_ethash_lean():
    """The same Ethash search as gen_ethash (identical outputs), laid out for memory-level
    parallelism: the DAG walk of an 8-lane group's 8 nonces keeps only the mixes in registers
    (lane j: words 4j..4j+3 of each, 32 registers); pages land in a per-thread shared ring through
    16-byte cp.async copies (no register per page in flight) and the Keccak-512 seed waits in
    shared memory (stride TMAX+1: conflict-free owner writes and group reads) until the final
    Keccak-256. Block size = TMAX (the search may give its interval fewer threads)."""
    p = "eh"
    T = ETHASH_LEAN_TMAX
    S = T + 1
    s = Src()
    hp = ", ".join(f"int {p}_h{i}" for i in range(8))
    header(s, p, "ethash", """// Ethash-style hashimoto nonce search (ethminer analogue, PAPER.md:876-879), lean-register form.
// Generated by kernels/gen_crypto.py (HF_ETHASH_FORM=lean). seed = Keccak-512(header_hash[8 words] ||
// nonce as 64-bit LE); mix = seed repeated to 32 words; 64 rounds: page = fnv(i ^ seed[0],
// mix[i % 32]) % npages (ethminer's modulo walk; remu: the fnv word read as uint32),
// mix = fnv(mix, dag[page]) over the 128-byte page; cmix = 8-word fnv fold;
// result = Keccak-256(seed || cmix).
// B200 mechanics: every thread computes the two Keccaks of its own nonce and parks the seed in
// shared memory; the DAG walk of the 8 nonces of an 8-lane group is shared (lane j holds words
// 4j..4j+3 of the 8 mixes, the lane owning mix[i % 32] computes each page index and broadcasts
// it with one shfl.idx) and every round's 8 pages per lane are copied by 16-byte cp.async into a
// per-thread shared ring (8 x 16 B), so pages in flight cost no registers: the walk needs ~60
// registers instead of ~125, and twice the warps (pages in flight) fit per SM.
// Criterion/checksum word = result word 0 (little-endian). Any warp-multiple block size up to """ + str(T) + """
// works (tunable: the partition search sizes it against its partner).""",
           f"int {p}_cnt[], int {p}_chk[], int {p}_bmin[], int {p}_dag[], int {p}_rc[], {hp}, int {p}_npages, "
           f"int {p}_nonce0, int {p}_count, int {p}_target", T, fixed=False)
    s(f"shared int {p}_ring[{8 * T * 4}];")
    s(f"shared int {p}_seed[{16 * S}];")
    A = {(x, y): Lane(f"a{x}{y}l", f"a{x}{y}h") for x in range(5) for y in range(5)}
    names = []
    for x in range(5):
        for y in range(5):
            names += [f"a{x}{y}l", f"a{x}{y}h"]
    for x in range(5):
        names += [f"c{x}l", f"c{x}h"]
    names += ["dl", "dh"] + [f"cm{i}" for i in range(8)]
    names += [f"x{h}_{k}" for h in range(8) for k in range(4)] + [f"z{h}" for h in range(8)]
    names += [f"pg{h}" for h in range(8)] + ["q0", "q1", "q2", "q3", "bw", "cw", "r0", "lj", "gb", "valid", "nonce"]
    names += ["tl", "th", "ul", "uh"]
    decls(s, names)
    s("int tid = threadIdx.x;")
    s("int nthr = blockDim.x;")
    s("int best = 2147483647;")
    s("int cnt = 0;")
    s("int chk = 0;")
    s("int lane = tid % 32;")
    s("lj = lane % 8;")
    s("gb = tid - lj;")
    s(f"for (int n0 = blockIdx.x * nthr + (tid / 32) * 32; n0 < {p}_count; n0 = n0 + gridDim.x * nthr) {{")
    s.ind += 1
    s("valid = n0 + lane < " + f"{p}_count;")
    s(f"nonce = {p}_nonce0 + n0 + lane;")
    words = [f"{p}_h{i}" for i in range(8)] + ["nonce", "0", "0x00000001"] + ["0"] * 6 + ["0x80000000"]
    absorb_words(s, A, words)
    keccak_f(s, A, f"{p}_rc")
    for i in range(8):
        ln = A[(i % 5, i // 5)]
        s(f"{p}_seed[{2 * i * S} + tid] = {ln.lo};")
        s(f"{p}_seed[{(2 * i + 1) * S} + tid] = {ln.hi};")
    s("warp_sync();")
    # lane j of the group takes words 4(j % 4) .. 4(j % 4) + 3 of each of the 8 group seeds
    s("int wrow = (lj % 4) * 4;")
    for h in range(8):
        s(f"z{h} = {p}_seed[gb + {h}];")
        for k in range(4):
            s(f"x{h}_{k} = {p}_seed[(wrow + {k}) * {S} + gb + {h}];")
    s("for (int it = 0; it < 64; it = it + 4) {")
    s.ind += 1
    s("int owner = (it % 32) / 4;")
    for k in range(4):
        for h in range(8):
            s(f"pg{h} = ((it + {k}) ^ z{h}) * 16777619 ^ x{h}_{k};")
            bcast8(s, f"pg{h}", "owner")
            s(f"pg{h} = remu(pg{h}, {p}_npages) * 8 + lj;")
        for h in range(8):
            s(f"async_copy({p}_ring, {h * T} + tid, {p}_dag, pg{h});")
        s("async_wait();")
        for h in range(8):
            s(f"vload({p}_ring, {h * T} + tid, q0, q1, q2, q3);")
            for j in range(4):
                s(f"x{h}_{j} = x{h}_{j} * 16777619 ^ q{j};")
    s.ind -= 1
    s("}")
    # cmix word j of nonce h sits in lane j of the group; each lane collects its own nonce's 8
    for h in range(8):
        s(f"cw = ((x{h}_0 * 16777619 ^ x{h}_1) * 16777619 ^ x{h}_2) * 16777619 ^ x{h}_3;")
        for k in range(8):
            s("bw = cw;")
            bcast8(s, "bw", k)
            s(f"if (lj == {h}) {{")
            s(f"  cm{k} = bw;")
            s("}")
    words = [f"{p}_seed[{i * S} + tid]" for i in range(16)] + [f"cm{i}" for i in range(8)] + ["0x00000001"] + ["0"] * 8 + ["0x80000000"]
    absorb_words(s, A, words)
    s("warp_sync();")  # every lane read its seed before the next nonce batch overwrites it
    keccak_f(s, A, f"{p}_rc")
    s(f"r0 = {A[(0, 0)].lo};")
    s("if (valid) {")
    s("  chk = chk + r0;")
    s(f"  if (ltu(r0, {p}_target)) {{")
    s("    cnt = cnt + 1;")
    s("    best = min(best, nonce);")
    s("  }")
    s("}")
    s.ind -= 1
    s("}")
    s(f"atomic_add({p}_chk[0], chk);")
    s("if (cnt > 0) {")
    s(f"  atomic_add({p}_cnt[0], cnt);")
    s("}")
    tail(s, p)
    return s.text()


def gen_ethash_reg():
    global ETHASH_FORM
    form, ETHASH_FORM = ETHASH_FORM, "reg"
    try:
        return gen_ethash()
    finally:
        ETHASH_FORM = form


def gen_blake2b_addc():
    """BLAKE2b with every 64-bit add carried by MK+ addc (add.cc/addc): ~13 % faster alone than the
    ltu form but slower fused next to an ALU-bound partner (profiles/r01_probe_blake2b_carry.json),
    so it is a second member form: the unfused baselines run whichever form is faster alone, and
    the fused search tries both."""
    global ADD64
    mode, ADD64 = ADD64, "addc"
    try:
        return gen_blake2b()
    finally:
        ADD64 = mode


def main():
    out = os.path.join(HERE, "b200")
    for name, gen in (("sha256d", gen_sha256d), ("blake256", gen_blake256), ("blake2b", gen_blake2b),
                      ("blake2b_addc", gen_blake2b_addc), ("ethash", gen_ethash), ("ethash_reg", gen_ethash_reg)):
        with open(os.path.join(out, name + ".mk"), "w") as f:
            f.write(gen())
        print("wrote", name)


if __name__ == "__main__":
    main()
