"""Regenerate the golden fixtures from the UNMODIFIED reference (TEST INFRASTRUCTURE ONLY).

Runs oracle/_ref/mkfuse_ref (the reference library, /root/reference/proj/src, linked by
oracle/Makefile) — it needs /root/reference, so it runs in the build container, never on
the GPU box. Outputs (committed):
  corpus_sources.json  the reference corpus kernels/images + golden goto text (fixtures)
  corpus_emit.json     sha256 of `fuse` output for all 64 ordered corpus pairs x
                       {goto, structured} x {regcap off, auto}, plus the `fuse` report
                       (fuser.cpp:553-558, mkfuse.cpp:109-167)
  corpus_digests.json  FNV-1a digests (memimage.cpp:198-242) of run_functional for the
                       acceptance sweep: 28 pairs x 20 seeds, sequential and fused
                       (acceptance_main.cpp:136-168), plus every corpus kernel alone
  members.json         interpreter outputs for the B200 member kernels at parity sizes
                       (see make_members below)
Usage: python tests/golden/make_golden.py [corpus|members|all]
"""
import hashlib
import itertools
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
REF = os.path.join(ROOT, "oracle", "_ref", "mkfuse_ref")
CORPUS = "/root/reference/proj/corpus"
STEMS = ["vector_add", "strided_sum", "histogram", "batchnorm", "shuffle_reduce", "streamer", "hasher", "empty"]


def run(*args):
    r = subprocess.run([REF, *map(str, args)], capture_output=True, text=True)
    if r.returncode != 0:
        return {"error": r.stderr.strip()}
    return {"out": r.stdout}


def dims(stem):
    t = open(f"{CORPUS}/{stem}.mk").read()
    m = re.search(r"dims \((\d+), (\d+), (\d+)\)( fixed)?", t)
    return int(m[1]) * int(m[2]) * int(m[3]), m[4] is None


def partition_for(a, b):
    """acceptance_main.cpp:65-71"""
    d1, t1 = dims(a)
    d2, t2 = dims(b)
    if d1 + d2 <= 1024:
        return d1, d2
    if t1:
        return 1024 - d2, d2
    return d1, 1024 - d1


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def make_corpus():
    # The corpus kernels and images are the reference's own test vectors; they are stored
    # as fixture data so the GPU tests can run without /root/reference.
    sources = {"kernels": {s: open(f"{CORPUS}/{s}.mk").read() for s in STEMS},
               "images": {s: open(f"{CORPUS}/images/{s}.img").read() for s in STEMS},
               "golden_goto": open("/root/reference/proj/tests/golden/fused_batchnorm_histogram.cu").read()}
    with open(os.path.join(HERE, "corpus_sources.json"), "w") as f:
        json.dump(sources, f, indent=1, sort_keys=True)
    emit = {}
    for a, b in itertools.product(STEMS, STEMS):
        d1, d2 = partition_for(a, b)
        entry = {"d1": d1, "d2": d2}
        for style in ("goto", "structured"):
            for rc in ("off", "auto"):
                r = run("fuse", f"{CORPUS}/{a}.mk", f"{CORPUS}/{b}.mk", "--d1", d1, "--d2", d2,
                        "--style", style, "--regcap", rc)
                entry[f"{style}_{rc}"] = sha(r["out"]) if "out" in r else r
        r = run("fusereport", f"{CORPUS}/{a}.mk", f"{CORPUS}/{b}.mk", "--d1", d1, "--d2", d2, "--regcap", "auto")
        entry["report"] = r.get("out", r)
        emit[f"{a}+{b}"] = entry
    with open(os.path.join(HERE, "corpus_emit.json"), "w") as f:
        json.dump(emit, f, indent=1, sort_keys=True)

    dig = {"pairs": {}, "kernels": {}}
    for i, a in enumerate(STEMS):
        for b in STEMS[i + 1:]:
            d1, d2 = partition_for(a, b)
            mem = ["--mem", f"{CORPUS}/images/{a}.img", "--mem", f"{CORPUS}/images/{b}.img"]
            rows = {}
            for seed in range(1, 21):
                s = run("seq", f"{CORPUS}/{a}.mk", f"{CORPUS}/{b}.mk", "--d1", d1, "--d2", d2, *mem, "--seed", seed)
                fz = run("fused", f"{CORPUS}/{a}.mk", f"{CORPUS}/{b}.mk", "--d1", d1, "--d2", d2, *mem, "--seed", seed)
                rows[str(seed)] = {"sequential": s["out"].split()[-1], "fused": fz["out"].split()[-1]}
            dig["pairs"][f"{a}+{b}"] = {"d1": d1, "d2": d2, "seeds": rows}
    dig["images"] = {}
    for a in STEMS:
        rows = {}
        for seed in (None, 1, 5):
            extra = [] if seed is None else ["--seed", seed]
            r = run("run", f"{CORPUS}/empty.mk", "--mem", f"{CORPUS}/images/{a}.img", *extra)
            rows[str(seed)] = r["out"].split()[-1]
        dig["images"][a] = rows
    for a in STEMS:
        rows = {}
        for seed in range(1, 6):
            r = run("run", f"{CORPUS}/{a}.mk", "--mem", f"{CORPUS}/images/{a}.img", "--seed", seed)
            rows[str(seed)] = r["out"].split()[-1]
        dig["kernels"][a] = rows
    # reference numbers for the machine model (machine.cpp:236-283)
    dig["register_bound"] = {}
    for case in [(32, 896, 24, 128, 4096), (16, 512, 16, 512, 256), (16, 512, 16, 512, 60000),
                 (40, 768, 20, 256, 0), (64, 128, 8, 896, 1024)]:
        dig["register_bound"][",".join(map(str, case))] = int(run("regbound", *case)["out"])
    dig["occupancy"] = {}
    for case in [(64, 24576, 512), (32, 24576, 512), (21, 640, 1024), (255, 0, 256), (16, 98304, 32)]:
        dig["occupancy"][",".join(map(str, case))] = run("occupancy", *case).get("out", "").strip()
    with open(os.path.join(HERE, "corpus_digests.json"), "w") as f:
        json.dump(dig, f, indent=1, sort_keys=True)
    print("corpus fixtures written")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("corpus", "all"):
        make_corpus()
    if what in ("members", "all"):
        sys.path.insert(0, HERE)
        import make_members  # noqa: E402

        make_members.main()
