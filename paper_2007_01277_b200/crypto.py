"""Crypto member workloads (C3/C4): memory-image texts for the generated kernels
(kernels/gen_crypto.py). Header words and the synthetic Ethash DAG are seeded so every
run is reproducible; the nonce range is [nonce0, nonce0 + count)."""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

MEMBERS = {"sha256d": "sh", "blake256": "bl", "blake2b": "b2", "ethash": "eh"}
THREADS = {"sha256d": 512, "blake256": 512, "blake2b": 512, "ethash": 1024}
# member source files per kind: ethash.mk is the lean-register form (the fused member),
# ethash_reg.mk the register form (faster alone); blake2b.mk carries its 64-bit adds with ltu
# (compare + select: the select runs on the FMA pipe), blake2b_addc.mk with add.cc/addc (faster
# alone, all ALU). The bench's unfused baselines run each kind's fastest form alone; the fused
# search tries every form in FUSED_FORMS.
FORMS = {"sha256d": ["sha256d"], "blake256": ["blake256"], "blake2b": ["blake2b", "blake2b_addc"],
         "ethash": ["ethash", "ethash_reg"]}
FUSED_FORMS = {"sha256d": ["sha256d"], "blake256": ["blake256"], "blake2b": ["blake2b", "blake2b_addc"],
               "ethash": ["ethash"]}
FORM_THREADS = {"ethash_reg": 256}
# Genesis block header (Bitcoin), the SHA-256d known-answer vector, as 20 big-endian words.
GENESIS_HEADER = bytes.fromhex(
    "01000000" + "00" * 32 + "3ba3edfd7a7b12b27ac72c3e67768f617fc81bc3888a51323a9fb8aa4b1e5e4a"
    "29ab5f49ffff001d1dac2b7c")


KECCAK_RC = [0x0000000000000001, 0x0000000000008082, 0x800000000000808A, 0x8000000080008000,
             0x000000000000808B, 0x0000000080000001, 0x8000000080008081, 0x8000000000008009,
             0x000000000000008A, 0x0000000000000088, 0x0000000080008009, 0x000000008000000A,
             0x000000008000808B, 0x800000000000008B, 0x8000000000008089, 0x8000000000008003,
             0x8000000000008002, 0x8000000000000080, 0x000000000000800A, 0x800000008000000A,
             0x8000000080008081, 0x8000000000008080, 0x0000000080000001, 0x8000000080008008]


def header_words(seed: int, n: int = 20) -> List[int]:
    """Deterministic pseudo-random header words (splitmix64 stream, low 32 bits)."""
    out, s = [], seed
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        out.append((z ^ (z >> 31)) & 0xFFFFFFFF)
    return out


def i32(x: int) -> int:
    x &= 0xFFFFFFFF
    return x - (1 << 32) if x & 0x80000000 else x


@dataclass
class CryptoWorkload:
    kind: str
    image: str
    nonces: int
    dag_bytes: int = 0


def workload(kind: str, count: int, grid: int, nonce0: int = 0, target: int = 1 << 12,
             words: Optional[List[int]] = None, header_seed: int = 2024, npages: int = 1 << 10,
             dag_seed: int = 77) -> CryptoWorkload:
    p = MEMBERS[kind]
    if words is None:
        words = header_words(header_seed, 20)
    nh = 8 if kind == "ethash" else 19
    lines = [f"array {p}_cnt int32 1 zero", f"array {p}_chk int32 1 zero", f"array {p}_bmin int32 {grid} zero"]
    lines += [f"scalar {p}_h{i} int32 {i32(words[i])}" for i in range(nh)]
    lines += [f"scalar {p}_nonce0 int32 {i32(nonce0)}", f"scalar {p}_count int32 {count}",
              f"scalar {p}_target int32 {i32(target)}"]
    dag_bytes = 0
    if kind == "sha256d":  # powers of two for the FMA-pipe rotates (gen_crypto HF_SHA_PIPES=fma, not the default)
        lines.append(f"array {p}_pw int32 32 values " + " ".join(str(i32(1 << k)) for k in range(32)))
    if kind == "ethash":
        rc = []
        for r in KECCAK_RC:
            rc += [i32(r), i32(r >> 32)]
        lines += [f"array {p}_dag int32 {npages * 32} seed {dag_seed} range -2147483648 2147483647",
                  f"array {p}_rc int32 48 values " + " ".join(map(str, rc)),
                  f"scalar {p}_npages int32 {npages}"]
        dag_bytes = npages * 128
    return CryptoWorkload(kind, "\n".join(lines) + "\n", count, dag_bytes)
