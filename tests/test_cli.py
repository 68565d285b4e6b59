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
