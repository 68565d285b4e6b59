"""The CLI's device commands (simulate / search / profile) against the reference fixtures."""
import os
import subprocess

import pytest

from conftest import ROOT, golden

EXE = os.path.join(ROOT, "paper_2007_01277_b200", "bin", "hfuse")
D = golden("corpus_digests.json")


def write_corpus(corpus, tmp_path):
    for stem, text in corpus["kernels"].items():
        (tmp_path / f"{stem}.mk").write_text(text)
    for stem, text in corpus["images"].items():
        (tmp_path / f"{stem}.img").write_text(text)


def run(*args):
    return subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=600)


@pytest.mark.gpu
def test_simulate_sequential_digest_matches_reference(gpu, corpus, tmp_path):
    """`hfuse simulate --sequential` prints the same digest as `mkfuse simulate --sequential`."""
    write_corpus(corpus, tmp_path)
    rec = D["pairs"]["vector_add+strided_sum"]
    r = run("simulate", "--sequential", tmp_path / "vector_add.mk", tmp_path / "strided_sum.mk",
            "--mem", tmp_path / "vector_add.img", "--mem", tmp_path / "strided_sum.img", "--seed", 3)
    assert r.returncode == 0, r.stderr
    kv = dict(line.split(" = ") for line in r.stdout.strip().splitlines())
    assert kv["digest"] == rec["seeds"]["3"]["sequential"]
    assert float(kv["elapsed_us"]) > 0
    # the reference's keys, in its order (mkfuse.cpp:190-196 + exec.cpp:995-1007), from device
    # measurements: cycles from the graph-timed member launches, counters from one ncu pass
    keys = [line.split(" = ")[0] for line in r.stdout.strip().splitlines()]
    assert keys[:8] == ["k1_cycles", "k2_cycles", "elapsed_cycles", "issue_slot_utilization",
                        "meminst_stall_fraction", "achieved_occupancy", "spill_loads_stores", "digest"]
    c1, c2 = int(kv["k1_cycles"]), int(kv["k2_cycles"])
    assert c1 > 0 and c2 > 0 and int(kv["elapsed_cycles"]) == c1 + c2
    u = float(kv["issue_slot_utilization"])
    assert 0.0 < u < 1.0 and 0.0 < float(kv["achieved_occupancy"]) <= 1.0
    assert 0.0 <= float(kv["meminst_stall_fraction"]) <= 1.0 and int(kv["spill_loads_stores"]) == 0


@pytest.mark.gpu
def test_fused_structured_file_simulates_to_reference_digest(gpu, corpus, tmp_path):
    write_corpus(corpus, tmp_path)
    out = tmp_path / "f.mk"
    assert run("fuse", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--d1", 896, "--d2", 128,
               "--style", "structured", "-o", out).returncode == 0
    r = run("simulate", out, "--mem", tmp_path / "batchnorm.img", "--mem", tmp_path / "histogram.img")
    kv = dict(line.split(" = ") for line in r.stdout.strip().splitlines())
    assert kv["digest"] == "d447034bfbccdc7c"  # proj/README.md:98,103


@pytest.mark.gpu
def test_search_on_device_and_profile_command(gpu, corpus, tmp_path):
    write_corpus(corpus, tmp_path)
    trace = tmp_path / "t.csv"
    r = run("search", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--mem", tmp_path / "batchnorm.img",
            "--mem", tmp_path / "histogram.img", "--trace", trace, "--reps", 3)
    assert r.returncode == 0, r.stderr
    assert "evaluated = 14" in r.stdout
    rows = trace.read_text().splitlines()
    assert rows[0] == "d1,d2,reg_cap,cycles,occupancy,utilization,us" and len(rows) == 15
    # the reference's --profiler-cmd contract: goto candidate named <fused>_<d1>_<cap>_<n>.cu
    cand = tmp_path / "fused_batchnorm_histogram_896_32_0.cu"
    assert run("fuse", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--d1", 896, "--d2", 128,
               "-o", cand).returncode == 0
    p = run("profile", cand, "--mem", tmp_path / "batchnorm.img", "--mem", tmp_path / "histogram.img")
    assert p.returncode == 0, p.stderr
    first = p.stdout.split()[0]
    assert first.isdigit() and int(first) > 0


@pytest.mark.gpu
def test_search_with_model_prefilter(gpu, corpus, tmp_path):
    """`--prefilter 2`: the 7 partitions are ranked by the model (constituents timed alone), only
    2 of them are fused and timed (uncapped + r0 each), every trace row carries its prediction."""
    write_corpus(corpus, tmp_path)
    trace = tmp_path / "t.csv"
    r = run("search", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--mem", tmp_path / "batchnorm.img",
            "--mem", tmp_path / "histogram.img", "--trace", trace, "--reps", 3, "--prefilter", 2,
            "--prefilter-tol", 0)
    assert r.returncode == 0, r.stderr
    assert "evaluated = 4" in r.stdout
    rows = trace.read_text().splitlines()
    assert rows[0] == "d1,d2,reg_cap,cycles,occupancy,utilization,us,predicted_us" and len(rows) == 5
    assert all(float(row.split(",")[-1]) > 0 for row in rows[1:])
    hf = gpu
    img = hf.Image(corpus["images"]["batchnorm"]).merge(hf.Image(corpus["images"]["histogram"])).upload()
    res = hf.search(corpus["kernels"]["batchnorm"], corpus["kernels"]["histogram"], img, reps=3, prefilter=2,
                    prefilter_tol=0.0)
    assert sorted(res["model"]) == [128, 256, 384, 512, 640, 768, 896] and len(res["trace"]) == 4


@pytest.mark.gpu
def test_profile_command_with_sm100_candidates(gpu, corpus, tmp_path):
    """`search --style sm100 --profiler-cmd 'hfuse profile ...'`: the command receives sm100
    candidates (manifest + the register cap as __maxnreg__) and times each on the device; the
    fold picks a point of the same 14-row sweep."""
    write_corpus(corpus, tmp_path)
    trace = tmp_path / "t.csv"
    cmd = f"{EXE} profile --mem {tmp_path / 'batchnorm.img'} --mem {tmp_path / 'histogram.img'} --reps 3"
    r = run("search", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--style", "sm100",
            "--profiler-cmd", cmd, "--trace", trace, "-o", tmp_path / "best.cu")
    assert r.returncode == 0, r.stderr
    rows = trace.read_text().splitlines()
    assert len(rows) == 15 and all(int(row.split(",")[3]) > 0 for row in rows[1:])


@pytest.mark.gpu
def test_search_on_several_devices_and_baselines(gpu, corpus, tmp_path):
    """`search --gpus N` times the sweep's candidates on N devices at once (MultiDeviceBackend;
    here two workers on device 0 through the HFUSE_SEARCH_DEVICES test knob, the only GPU of the
    box): the same 14-point sweep and fold. `--baseline both` then times the unfused members
    sequentially and on two streams against the winner."""
    write_corpus(corpus, tmp_path)
    env = dict(os.environ, HFUSE_SEARCH_DEVICES="0,0")
    r = subprocess.run([EXE, "search", tmp_path / "batchnorm.mk", tmp_path / "histogram.mk", "--mem",
                        tmp_path / "batchnorm.img", "--mem", tmp_path / "histogram.img", "--reps", "5",
                        "--baseline", "both"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr
    kv = dict(line.split(" = ") for line in r.stdout.strip().splitlines() if " = " in line)
    assert kv["devices"] == "2" and kv["evaluated"] == "14"
    assert float(kv["best_us"]) > 0 and float(kv["sequential_us"]) > 0 and float(kv["two_stream_us"]) > 0
    assert abs(float(kv["speedup"]) - min(float(kv["sequential_us"]), float(kv["two_stream_us"])) /
               float(kv["best_us"])) < 1e-3
