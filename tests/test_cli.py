"""The hfuse CLI as a drop-in for `mkfuse` (tools/mkfuse.cpp): flags, stdout keys, exit codes."""
import os
import subprocess

from conftest import ROOT, golden

EXE = os.path.join(ROOT, "paper_2007_01277_b200", "bin", "hfuse")
EMIT = golden("corpus_emit.json")


def run(*args, cwd=None):
    return subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, cwd=cwd)


def write_corpus(corpus, tmp_path):
    for stem, text in corpus["kernels"].items():
        (tmp_path / f"{stem}.mk").write_text(text)
    for stem, text in corpus["images"].items():
        (tmp_path / f"{stem}.img").write_text(text)


def test_fuse_matches_reference_report_and_file(corpus, tmp_path):
    write_corpus(corpus, tmp_path)
    out = tmp_path / "fused.cu"
    r = run("fuse", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--d1", 896, "--d2", 128,
            "--style", "goto", "-o", out)
    assert r.returncode == 0
    assert r.stdout == EMIT["batchnorm+histogram"]["report"] + f"wrote {out}\n"
    assert out.read_text() == corpus["golden_goto"]


def test_errors_exit_1_with_position(corpus, tmp_path):
    (tmp_path / "bad.mk").write_text("kernel k() dims (32, 1, 1) {\n  y = 1;\n}\n")
    write_corpus(corpus, tmp_path)
    r = run("fuse", tmp_path / "bad.mk", tmp_path / "histogram.mk", "--d1", 32, "--d2", 128)
    assert r.returncode == 1 and r.stderr.strip() == "error[UnknownIdentifier] 2:3: unknown identifier 'y'"
    r = run("fuse", tmp_path / "missing.mk", tmp_path / "histogram.mk", "--d1", 32, "--d2", 128)
    assert r.returncode == 1 and r.stderr.startswith("error[Io]")


def test_occupancy_and_check(corpus, tmp_path):
    r = run("occupancy", "--regs", 64, "--shmem", 24576, "--threads", 512)
    assert r.stdout.splitlines()[:2] == ["blocks_per_sm = 2", "limiting_resource = registers"]
    write_corpus(corpus, tmp_path)
    assert run("check", tmp_path / "histogram.mk").stdout.startswith("ok: 1 kernel(s), 1 function(s)")


def test_search_with_profiler_command(corpus, tmp_path):
    write_corpus(corpus, tmp_path)
    trace = tmp_path / "t.csv"
    r = run("search", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--profiler-cmd", "echo 11",
            "--trace", trace, "-o", tmp_path / "w.mk")
    assert r.returncode == 0 and "evaluated = 14" in r.stdout and "best_d1 = 128" in r.stdout
    assert len(trace.read_text().splitlines()) == 15
    assert run("check", tmp_path / "w.mk").returncode == 0


def test_lower_and_emit(tmp_path):
    from paper_2007_01277_b200 import pairs
    p = tmp_path / "h.mk"
    p.write_text(pairs.source("b200", "histogram"))
    low = run("lower", p)
    assert low.returncode == 0 and "vload" not in low.stdout and "__vx0" in low.stdout
    em = run("emit", p)
    assert em.returncode == 0 and "reinterpret_cast<const float4*>(hi_x)" in em.stdout


def test_fuse_interval_register_budgets(tmp_path):
    """B200 extension: `--interval-regs R1,R2` emits __maxnreg__(pool) and one setmaxnreg per
    interval; misaligned partitions, bad budgets, oversized pools and --regcap are rejected."""
    k = os.path.join(ROOT, "paper_2007_01277_b200", "kernels", "b200")
    bl, eh = os.path.join(k, "blake256.mk"), os.path.join(k, "ethash.mk")
    out = tmp_path / "f.cu"
    r = run("fuse", bl, eh, "--d1", 512, "--d2", 384, "--style", "sm100", "--sm", "b200",
            "--interval-regs", "32,120", "-o", out)
    assert r.returncode == 0, r.stderr
    assert "interval_regs = 32,120 (launch 72)" in r.stdout
    text = out.read_text()
    assert "__maxnreg__(72)" in text and "__launch_bounds__" not in text
    assert text.count("setmaxnreg.dec.sync.aligned.u32 32;") == 1
    assert text.count("setmaxnreg.inc.sync.aligned.u32 120;") == 1
    assert text.index("setmaxnreg.dec") < text.index("setmaxnreg.inc")
    for args, code in [(("--d1", 512, "--d2", 320, "--interval-regs", "32,120"), "InvalidArgument"),
                       (("--d1", 512, "--d2", 384, "--interval-regs", "30,120"), "InvalidArgument"),
                       (("--d1", 512, "--d2", 384, "--interval-regs", "64,128"), "DoesNotFit"),
                       (("--d1", 512, "--d2", 384, "--interval-regs", "32,120", "--regcap", "64"),
                        "InvalidArgument"),
                       (("--d1", 512, "--d2", 384, "--interval-regs", "32,120", "--style", "goto"),
                        "InvalidArgument")]:
        style = [] if "--style" in args else ["--style", "sm100"]
        r = run("fuse", bl, eh, *args, *style, "--sm", "b200", "-o", out)
        assert r.returncode == 1 and r.stderr.startswith(f"error[{code}]"), (args, r.stderr)


def test_search_sweeps_interval_budgets_with_profiler_command(tmp_path):
    """`search --budgets`: warpgroup-aligned partitions also get per-interval register budget
    candidates (trace reg_cap column `R1/R2`), handed to the command as sm100 text."""
    k = os.path.join(ROOT, "paper_2007_01277_b200", "kernels", "b200")
    trace = tmp_path / "t.csv"
    prof = tmp_path / "prof.sh"
    prof.write_text("#!/bin/sh\nif grep -q setmaxnreg \"$1\"; then echo 5; else echo 11; fi\n")
    prof.chmod(0o755)
    r = run("search", os.path.join(k, "blake256.mk"), os.path.join(k, "ethash.mk"), "--d0", 896, "--budgets",
            "--profiler-cmd", prof, "--trace", trace, "-o", tmp_path / "w.cu", "--style", "sm100")
    assert r.returncode == 0, r.stderr
    rows = [line.split(",") for line in trace.read_text().splitlines()[1:]]
    budgets = [row[2] for row in rows if "/" in row[2]]
    assert budgets and all(row[3] == "5" for row in rows if "/" in row[2])
    assert "best_interval_regs = " + budgets[0] in r.stdout
    assert "setmaxnreg" in (tmp_path / "w.cu").read_text()


def test_prefilter_needs_a_measuring_backend(corpus, tmp_path):
    """The model pre-filter times constituents alone; a profiler command cannot, so the sweep
    stays exhaustive (the reference's 14 points)."""
    write_corpus(corpus, tmp_path)
    r = run("search", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--profiler-cmd", "echo 11",
            "--prefilter", 2)
    assert r.returncode == 0 and "evaluated = 14" in r.stdout


def test_sm100_export_carries_cap_and_manifest(corpus, tmp_path):
    """`fuse --style sm100 --regcap 32`: the cap is in the code as __maxnreg__(32) (nvcc ignores
    --maxrregcount under __launch_bounds__) and the first line is the manifest `hfuse profile`
    rebuilds the launch from (the exported text used to drop the cap)."""
    for stem in ("batchnorm", "histogram"):
        (tmp_path / f"{stem}.mk").write_text(corpus["kernels"][stem])
    out = tmp_path / "f.cu"
    r = subprocess.run([EXE, "fuse", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--d1", "896", "--d2",
                        "128", "--style", "sm100", "--regcap", "32", "-o", out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    text = out.read_text()
    first = text.splitlines()[0]
    assert first.startswith("// hfuse-sm100 entry=fused_batchnorm_histogram threads=1024 ")
    assert "params=" in first and "__maxnreg__(32)" in text and "__launch_bounds__" not in text
