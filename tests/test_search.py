"""Partition search (search.cpp:66-188) through the external-command profiler backend,
the reference's only process boundary (mkfuse search --profiler-cmd), on CPU."""
import os
import stat

import pytest


def test_trace_shape_and_tie_break(hf, corpus):
    """BN+Hist at d0=1024: 7 partitions x {uncapped, r0} = 14 rows (test_search.cpp:22-49);
    a constant profiler ties everywhere -> smallest d1, no cap (search.cpp:72-89)."""
    r = hf.search(corpus["kernels"]["batchnorm"], corpus["kernels"]["histogram"], profiler_cmd="echo 4242 ;true")
    assert len(r["trace"]) == 14
    assert [t["d1"] for t in r["trace"]] == [d for d in range(128, 1024, 128) for _ in (0, 1)]
    assert (r["d1"], r["d2"], r["reg_cap"], r["best_time"]) == (128, 896, None, 4242)
    assert r["trace_csv"].startswith("d1,d2,reg_cap,cycles,occupancy,utilization\n")


def test_argmin_over_a_scripted_profiler(hf, corpus, tmp_path):
    """The profiler sees `<name>_<d1>_<regcap|0>_<n>.cu` (search.cpp:35-39); cost = |d1 - 640|
    + (cap ? 1 : 0) makes (640, no cap) the unique minimum."""
    script = tmp_path / "prof.sh"
    script.write_text('#!/bin/sh\nb=$(basename "$1" .cu)\nd1=$(echo $b | awk -F_ \'{print $(NF-2)}\')\n'
                      'cap=$(echo $b | awk -F_ \'{print $(NF-1)}\')\n'
                      'c=$(( (d1 > 640 ? d1 - 640 : 640 - d1) * 10 + (cap > 0 ? 1 : 0) + 5 ))\necho $c\n')
    script.chmod(script.stat().st_mode | stat.S_IEXEC)
    r = hf.search(corpus["kernels"]["batchnorm"], corpus["kernels"]["histogram"], profiler_cmd=str(script))
    assert (r["d1"], r["reg_cap"], r["best_time"]) == (640, None, 5)
    assert min(t["cycles"] for t in r["trace"]) == r["best_time"]


def test_fixed_pair_evaluates_one_partition(hf, corpus):
    r = hf.search(corpus["kernels"]["streamer"], corpus["kernels"]["hasher"], profiler_cmd="echo 7")
    assert len(r["trace"]) == 2 and (r["d1"], r["d2"]) == (512, 512)
    assert r["trace"][0]["reg_cap"] == "none" and r["trace"][1]["reg_cap"] != "none"


def test_small_d0(hf, corpus):
    r = hf.search(corpus["kernels"]["vector_add"], corpus["kernels"]["strided_sum"], d0=256, profiler_cmd="echo 1")
    assert len(r["trace"]) == 2 and r["d1"] == 128


def test_infeasible_everywhere(hf):
    k = "kernel a(int x[]) dims (64, 1, 1) { x[0] = 1; }"
    g = "//@ grid=3\nkernel b(int y[]) dims (64, 1, 1) { y[0] = 1; }"
    with pytest.raises(hf.HFuseError) as e:
        hf.search(k, g, profiler_cmd="echo 1")
    assert e.value.name == "NothingFeasible"
