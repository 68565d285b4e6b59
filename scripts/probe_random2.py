"""Random 128-byte page reads over the Ethash bench DAG (33,554,393 pages, 4.3 GB, prime count,
modulo walk): the HBM random-page ceiling with well-mixed (murmur-finalized) page indices,
independent chains (`chains` pages in flight per lane) vs data-dependent chains (the next page
index folds the loaded words, as in Ethash). Diagnostic: profiles/r02_probe_random2.jsonl."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402

NPAGES = 33554393
ROUNDS = 64


def source(chains, threads, dependent):
    decl = " ".join(f"int a{c}; int x{c};" for c in range(chains))
    init = "\n".join(f"    x{c} = g * {chains} + {c};" for c in range(chains))
    body = []
    for c in range(chains):
        mix = f"x{c}" if dependent else f"(g * {chains} + {c})"
        body.append(f"      h = ({mix} ^ (r * 0x85ebca77)) * 0x2c1b3c6d;")
        body.append("      h = (h ^ shr_u(h, 15)) * 0x297a2d39;")
        body.append("      h = h ^ shr_u(h, 13);")
        body.append(f"      a{c} = warp_bcast(h, 0, 8);")
        body.append(f"      a{c} = remu(a{c}, npages) * 8 + lj;")
    for c in range(chains):
        body.append(f"      vload(dag, a{c}, q0, q1, q2, q3);")
        body.append(f"      x{c} = (x{c} * 16777619) ^ q0 ^ q1 ^ q2 ^ q3;")
    fold = " ^ ".join(f"x{c}" for c in range(chains))
    return f"""kernel rnd(int dag[], int sink[], int npages, int groups) dims ({threads}, 1, 1) {{
  int nthr = blockDim.x;
  int lj = threadIdx.x % 8;
  int h; int q0; int q1; int q2; int q3; int acc = 0; {decl}
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
    img = hf.Image(f"array dag int32 {NPAGES * 32} seed 7 range -2147483648 2147483647\n"
                   f"array sink int32 4 zero\nscalar npages int32 {NPAGES}\nscalar groups int32 {1 << 17}\n").upload()
    for dependent in (False, True):
        for chains in (1, 2, 4, 8):
            for threads, grid in ((256, 1184), (512, 592), (1024, 296)):
                try:
                    m = hf.Module.kernel(source(chains, threads, dependent), grid=grid, specialize=img)
                except hf.HFuseError as e:
                    print(json.dumps({"chains": chains, "err": str(e)[:200]}), flush=True)
                    continue
                t = hf.time_graph("single", m, None, img, grid, 0, reps=3, samples=3)["mean_us"]
                nbytes = (1 << 17) * ROUNDS * chains * 128
                print(json.dumps({"dependent": dependent, "chains": chains, "threads": threads, "grid": grid,
                                  "regs": m.info.regs, "bps": m.info.blocks_per_sm, "us": round(t, 1),
                                  "gbs": round(nbytes / (t * 1e3), 1)}), flush=True)


if __name__ == "__main__":
    main()
