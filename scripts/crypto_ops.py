"""Algorithmic per-nonce operation counts of the crypto members, counted from their kernel
SOURCE (paper_2007_01277_b200/kernels/b200/*.mk) -> profiles/crypto_ops.json.

SURVEY.md §8d defines the issue-rate roofline of a hash as sum(warp instructions) /
(148 SMs x 4 schedulers x f_clk) with "per-nonce 32-bit integer op counts derived from the
builder's kernel source and committed as a table". This script is that table: it walks the
per-nonce loop body of each generated member (straight-line MK+ code, inner loops with
constant trip counts multiplied out) and counts one operation per source-level 32-bit operation
-- every binary/unary operator, every builtin call (rotr, rotl, shr_u, fshr, fshl, ltu, min,
max, int_rz, warp_bcast, warp_shfl_xor, atomic_add) and every array access (one per element
for vload/vstore). Assignments, declarations and literal signs are free. The count is fixed by
the algorithm as written, independent of what nvcc emits for any fused or unfused kernel, so a
slower kernel cannot raise its own ceiling.

Per nonce: a thread of SHA-256d / BLAKE-256 / BLAKE2b hashes one nonce per loop iteration; an
Ethash thread runs its own nonce's two Keccaks plus its lane's share of its 8-lane group's DAG
walk per iteration (8 nonces per group, so the count per iteration is the count per nonce).
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = os.path.join(ROOT, "paper_2007_01277_b200", "kernels", "b200")
MEMBERS = ("sha256d", "blake256", "blake2b", "ethash")
CALLS = ("rotr", "rotl", "shr_u", "fshr", "fshl", "ltu", "min", "max", "int_rz", "warp_bcast",
         "warp_shfl_xor", "atomic_add", "addc")
FOR_RE = re.compile(r"for \(int (\w+) = (-?\d+); \1 < (\w+); \1 = \1 \+ (\d+)\) \{")
NONCE_RE = re.compile(r"for \(int (n|n0) = blockIdx\.x")


def line_ops(line: str) -> int:
    s = line.split("//")[0].strip()
    if not s or s in ("{", "}", "} else {") or s.startswith(("int ", "float ", "shared ")) and "=" not in s:
        return 0
    if s.startswith("int ") or s.startswith("float "):
        s = s.split(" ", 1)[1]  # declaration with initializer: count the initializer
    n = 0
    m = re.match(r"vload\(\w+, (.*), \w+, \w+, \w+, \w+\);", s)
    if m:  # a 128-bit load: the index expression + 4 element loads
        return line_ops(m.group(1) + ";") + 4
    for c in CALLS:
        n += len(re.findall(r"\b%s\(" % c, s))
    n += len(re.findall(r"\[", s))                         # array element accesses
    t = re.sub(r"(?<=[(,=])\s*-\s*(?=\d)", "", s)          # literal signs
    t = re.sub(r"\b0x[0-9a-fA-F]+\b|\b\d+\b", "0", t)
    t = t.replace("if (", "(").replace("while (", "(")
    n += len(re.findall(r"<<|>>|<=|>=|==|!=|&&|\|\||[-+*/%^&|<>!~]", t.split("=", 1)[1] if re.match(r"^\w+(\[.*\])? = ", t) else t))
    return n


def count(path: str) -> dict:
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if NONCE_RE.search(ln))
    depth0 = lines[start].index("for")
    total, stack = 0, [1]   # multiplier stack of the enclosing constant-trip loops
    i = start + 1
    while i < len(lines):
        ln = lines[i]
        ind = len(ln) - len(ln.lstrip())
        s = ln.strip()
        if s == "}" and ind == depth0:
            break                                          # end of the nonce loop
        m = FOR_RE.search(s)
        if m:
            lo, hi, step = int(m.group(2)), m.group(3), int(m.group(4))
            trips = (int(hi) - lo + step - 1) // step if hi.isdigit() else None
            if trips is None:
                raise ValueError(f"{path}:{i + 1}: loop bound {hi} is not a constant")
            total += stack[-1] * trips * 2                 # compare + increment per trip
            stack.append(stack[-1] * trips)
        elif s.endswith("{"):
            total += stack[-1] * line_ops(s[:-1])          # if / while condition
            stack.append(stack[-1])
        elif s.startswith("}"):
            stack.pop()
            if s.endswith("{"):                            # } else {
                stack.append(stack[-1])
        else:
            total += stack[-1] * line_ops(s)
        i += 1
    return {"ops_per_nonce": total, "source": os.path.relpath(path, ROOT),
            "loop_line": start + 1}


def main():
    out = {k: count(os.path.join(KERNELS, k + ".mk")) for k in MEMBERS}
    out["_rule"] = ("one op per source-level 32-bit operation of the per-nonce loop body (operators, builtin "
                    "calls, array element accesses), constant-trip inner loops multiplied out; "
                    "issue time = nonces x ops / 32 / (148 x 4 x f_sm) (SURVEY.md §8d)")
    dst = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "crypto_ops.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    for k in MEMBERS:
        print(k, out[k]["ops_per_nonce"])


if __name__ == "__main__":
    main()
