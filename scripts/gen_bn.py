"""BatchNorm-statistics member with K 128-bit loads in flight per thread (kernels/b200/batchnorm.mk
is K = 4 at 1024 threads). The per-channel block form of batchnorm.mk fills 256 of the B200's 296
block slots at C = 256, so its loads in flight (not its bytes) bound it: more loads per thread
raise the bytes in flight per block. Used by scripts/probe_bn_mlp.py."""


def gen_bn(K: int, threads: int = 1024) -> str:
    src = open(__file__.replace("scripts/gen_bn.py", "paper_2007_01277_b200/kernels/b200/batchnorm.mk")).read()
    head, rest = src.split("  float v0;", 1)
    head = head.replace("dims (1024, 1, 1)", f"dims ({threads}, 1, 1)")
    tail = rest[rest.index("    while (j < total4) {"):]
    vs = " ".join(f"float v{i};" for i in range(4 * K))
    out = [head.rstrip("\n"), "  " + vs, "  float e0; float e1; float e2; float e3;",
           "  float avg; float m2; int n; float o_avg; float o_m2; int o_n; int tot; float fac; float delta;",
           "  for (int c = blockIdx.x; c < bn_C; c = c + gridDim.x) {",
           "    n = 0;", "    float K = 0.0;", "    float s1 = 0.0;", "    float s2 = 0.0;",
           "    int total4 = bn_N * hw4;", "    if (tid < total4) {", "      int b0 = tid / hw4;",
           "      K = bn_x[((b0 * bn_C + c) * hw4 + tid - b0 * hw4) * 4];", "    }", "    int j = tid;",
           f"    while (j + {K - 1} * nthr < total4) {{"]
    for i in range(K):
        off = "" if i == 0 else (" + nthr" if i == 1 else f" + {i} * nthr")
        out.append(f"      int p{i} = (j{off}) / hw4;")
    for i in range(K):
        off = "" if i == 0 else (" + nthr" if i == 1 else f" + {i} * nthr")
        out.append(f"      vload(bn_x, (p{i} * bn_C + c) * hw4 + j{off} - p{i} * hw4, v{4*i}, v{4*i+1}, v{4*i+2}, v{4*i+3});")
    for i in range(K):
        for q in range(4):
            out.append(f"      e{q} = v{4*i+q} - K;")
        out.append("      s1 = s1 + ((e0 + e1) + (e2 + e3));")
        out.append("      s2 = s2 + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));")
    out.append(f"      n = n + {4 * K};")
    out.append(f"      j = j + {K} * nthr;")
    out.append("    }")
    return "\n".join(out) + "\n" + tail
