"""TEST INFRASTRUCTURE ONLY: the parity checker for device outputs of the DL members and the
crypto members, used by tests/ and by bench.py's cpu_baseline leg (outside every timed region)
to check the exact fused kernels the bench times.

Expected outputs come from the C restatement (hf_oracle.c, pinned on the reference interpreter
by tests/test_oracle.py) on the same seeded inputs, and from crypto_ref (pinned on the standard
test vectors by tests/test_crypto.py). Rules (/root/reference/proj/tests/
test_fuser.cpp:459 form): bit-exact for Hist, MaxPool values and indices, Upsample, Im2Col and
every crypto output; BatchNorm mean and biased variance within 1e-5 * max(1, |x|) of fp64.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle

BN_TOL = 1e-5


def member_expected(key: str, image_text: str) -> dict:
    """The member's expected outputs for a workload image (memimage text of pairs.py)."""
    a, s = oracle.parse_image(image_text)
    s = {k: (int(v) if not isinstance(v, np.floating) else float(v)) for k, v in s.items()}
    if key == "bn":
        mean, var = oracle.bn_stats(a["bn_x"], s["bn_N"], s["bn_C"], s["bn_HW"])
        return {"mean": mean, "var": var}
    if key == "hist":
        return {"hi_out": oracle.hist(a["hi_x"])}
    if key == "maxpool":
        y, idx = oracle.maxpool(a["mp_x"], s["mp_NC"], s["mp_H"], s["mp_W"])
        return {"mp_y": y, "mp_idx": idx}
    if key == "upsample":
        return {"us_y": oracle.upsample(a["us_x"], s["us_NC"], s["us_IH"], s["us_IW"])}
    if key == "im2col":
        return {"ic_col": oracle.im2col(a["ic_x"], s["ic_NC"], s["ic_H"], s["ic_W"])}
    raise KeyError(key)


def bn_within_tol(got_stats: np.ndarray, mean: np.ndarray, var: np.ndarray, tol: float = BN_TOL):
    """(ok, worst relative error) of float32 (mean, var) pairs against fp64."""
    got = np.asarray(got_stats, np.float32).reshape(-1, 2).astype(np.float64)
    err = 0.0
    ok = True
    for col, want in ((0, mean), (1, var)):
        d = np.abs(got[:, col] - want) / np.maximum(1.0, np.abs(want))
        err = max(err, float(d.max()))
        ok &= bool(np.all(d <= tol))
    return ok, err


def check_member(key: str, get, expected: dict) -> dict:
    """Compare device outputs (get(name) -> numpy array) with `expected`.
    Returns {"ok": bool, "what": ..., "max_rel_err" (BN) or "mismatches": count}."""
    if key == "bn":
        ok, err = bn_within_tol(get("bn_stats"), expected["mean"], expected["var"])
        return {"ok": ok, "what": "bn mean/var vs fp64, rel tol 1e-5", "max_rel_err": err}
    bad = 0
    for name, want in expected.items():
        got = get(name)
        if got.shape != want.shape:
            return {"ok": False, "what": f"{name} shape {got.shape} != {want.shape}", "mismatches": -1}
        bad += int(np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)))
    return {"ok": bad == 0, "what": "bit-exact " + "+".join(expected), "mismatches": bad}


def crypto_expected(kind: str, count: int, grid: int, nonce0: int, target: int, threads: int,
                    npages: int, words=None) -> dict:
    """crypto_ref.search_outputs for the nonce sub-range, the block assignment of `grid` blocks
    of `threads` lanes of this member's interval, and the workload's seeded DAG."""
    from oracle import crypto_ref as C
    from paper_2007_01277_b200 import crypto
    words = words or crypto.header_words(2024, 20)
    dag = C.LazyDag(77, npages) if kind == "ethash" else None
    return C.search_outputs(kind, words, nonce0, count, target, grid, threads, dag=dag, n_pages=npages)
