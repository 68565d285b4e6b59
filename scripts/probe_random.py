"""Random 128-byte page reads from a 4 GiB array (the Ethash DAG access pattern): each 8-lane
group reads `chains` independent pseudo-random pages per round (group-uniform addresses, one
coalesced 128-B segment per page), so the result is the HBM random-page ceiling for a given
number of pages in flight. Diagnostic (results: profiles/r01_probe_random_pages.jsonl)."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402

NPAGES = 1 << 25  # 4 GiB of 128-B pages
ROUNDS = 64


def source(chains, threads):
    decl = " ".join(f"int a{c}; int x{c};" for c in range(chains))
    init = "\n".join(f"    x{c} = g * {chains} + {c};" for c in range(chains))
    body = []
    for c in range(chains):
        seed = f"(g * {chains} + {c})"
        body.append(f"      a{c} = ((r ^ {seed}) * 16777619 + {seed} * 40503) & (npages - 1);")
    for c in range(chains):
        body.append(f"      vload(dag, a{c} * 8 + lj, q0, q1, q2, q3);")
        body.append(f"      x{c} = (x{c} * 16777619) ^ q0 ^ q1 ^ q2 ^ q3;")
    fold = " ^ ".join(f"x{c}" for c in range(chains))
    return f"""kernel rnd(int dag[], int sink[], int npages, int groups) dims ({threads}, 1, 1) {{
  int nthr = blockDim.x;
  int lj = threadIdx.x % 8;
  int q0; int q1; int q2; int q3; int acc = 0; {decl}
  for (int g = (blockIdx.x * nthr + threadIdx.x) / 8; g < groups; g = g + gridDim.x * nthr / 8) {{
{init}
    for (int r = 0; r < {ROUNDS}; r = r + 1) {{
""" + "\n".join(body) + f"""
    }}
    acc = acc ^ {fold};
  }}
  if (acc == 123456789) {{
    sink[0] = acc;
  }}
}}
"""


def main():
    groups = 1 << 17  # 131072 groups x ROUNDS x chains pages
    img = hf.Image(f"array dag int32 {NPAGES * 32} seed 7 range -2147483648 2147483647\n"
                   f"array sink int32 4 zero\nscalar npages int32 {NPAGES}\nscalar groups int32 {groups}\n").upload()
    for chains in (1, 4, 8, 16):
        for threads, grid in ((256, 296), (256, 1184), (1024, 296)):
            m = hf.Module.kernel(source(chains, threads), grid=grid, specialize=img)
            t = hf.time("single", m, None, img, grid, warmup=1, reps=5)["iqm_us"]
            nbytes = groups * ROUNDS * chains * 128
            print(json.dumps({"dependent": False, "chains": chains, "threads": threads, "grid": grid,
                              "regs": m.info.regs, "us": round(t, 1), "gbs": round(nbytes / (t * 1e3), 1)}),
                  flush=True)


if __name__ == "__main__":
    main()
