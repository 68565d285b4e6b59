"""Hist member with K 128-bit loads in flight per thread (kernels/b200/histogram.mk is K = 4):
the same warp-private shared-memory bins and tail handling, K vector loads issued before any
binning. Used by scripts/probe_hist_mlp.py."""


def gen_hist(K: int, threads: int = 1024) -> str:
    src = open(__file__.replace("scripts/gen_hist.py", "paper_2007_01277_b200/kernels/b200/histogram.mk")).read()
    head, rest = src.split("  float v0;", 1)
    head = head.replace("dims (1024, 1, 1)", f"dims ({threads}, 1, 1)")
    tail = rest[rest.index("  // the n % 4 trailing values"):]
    vs = " ".join(f"float v{i};" for i in range(4 * K))
    out = [head.rstrip("\n"), "  " + vs,
           f"  for (int i = blockIdx.x * nthr + tid; i < n4; i = i + {K} * stride) {{"]
    for k in range(1, K):
        out.append(f"    int j{k} = {'i' if k == 1 else f'j{k - 1}'} + stride;")
    out.append("    vload(hi_x, i, v0, v1, v2, v3);")
    for k in range(1, K):
        out.append(f"    vload(hi_x, min(j{k}, last), v{4 * k}, v{4 * k + 1}, v{4 * k + 2}, v{4 * k + 3});")
    for k in range(K):
        ind = "    "
        if k:
            out.append(f"    if (j{k} < n4) {{")
            ind = "      "
        for q in range(4):
            v = f"v{4 * k + q}"
            out.append(f"{ind}if ({v} >= -4.0 && {v} <= 4.0) {{")
            out.append(f"{ind}  atomic_add(hi_bins[wb + min(int_rz(({v} + 4.0) * 8.0), 63)], 1);")
            out.append(f"{ind}}}")
        if k:
            out.append("    }")
    out.append("  }")
    return "\n".join(out) + "\n" + tail


if __name__ == "__main__":
    import sys
    print(gen_hist(int(sys.argv[1]) if len(sys.argv) > 1 else 4))
