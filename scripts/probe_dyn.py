"""Probe: dynamic interval scheduling (hf_build_fused_opts vgrid) vs the static partition for
DL pairs at C2 sizes. For every pair: the static best of profiles/r02_bench_detail.json re-timed,
two-stream at its grids, and a sweep of dynamic variants: d0 in {1024, 512} (persistent grid =
148 x 2048/d0), splits in steps of 128, virtual-block sizes (bytes per virtual block) for the
grid-stride members (BatchNorm keeps one channel per virtual block). Graph protocol.
Output: JSON lines on stdout."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402


def vgrid_of(key, work, vb_bytes):
    if key == "bn":
        return int(work.image.split("scalar bn_C int32 ")[1].split()[0])
    return max(148, work.bytes // vb_bytes)


def main():
    pairs = [tuple(p.split("+")) for p in (sys.argv[1] if len(sys.argv) > 1 else
                                          "bn+im2col,im2col+upsample,maxpool+upsample,bn+upsample,hist+im2col").split(",")]
    vbs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "131072,524288,2097152").split(",")]
    detail = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_detail.json")))
    static = {r["pair"]: r for r in detail["results"]}
    import torch
    stream = torch.cuda.current_stream()
    for a, b in pairs:
        wa, wb = P.MEMBERS[a].sizes["full"](), P.MEMBERS[b].sizes["full"]()
        sa, sb = P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem)
        img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload(stream)
        st = static[f"{a}+{b}"]
        ms = hf.Module.fused(sa, sb, st["d1"], st["d2"], regcap=st["reg_cap"] or "off", grid=st["grid"], specialize=img)
        t_static = hf.time_graph("single", ms, None, img, st["grid"], 0, reps=20, samples=5, stream=stream)
        ka = hf.Module.kernel(sa, grid=296, specialize=img)
        kb = hf.Module.kernel(sb, grid=296, specialize=img)
        ga, gb = st["two_stream_grids"]
        t_two = hf.time_graph("two_stream", ka, kb, img, ga, gb, reps=20, samples=5, stream=stream)
        print(json.dumps({"pair": f"{a}+{b}", "static_us": round(t_static["mean_us"], 2),
                          "two_stream_us": round(t_two["mean_us"], 2), "static_cfg": [st["grid"], st["d1"], st["reg_cap"]]}),
              flush=True)
        best = None
        for d0 in (1024, 512):
            grid = 148 * (2048 // d0)
            for d1 in range(128, d0, 128):
                for vb in vbs:
                    v1, v2 = vgrid_of(a, wa, vb), vgrid_of(b, wb, vb)
                    for cap in ("off", 32):
                        try:
                            m = hf.Module.fused_opts(sa, sb, d1, d0 - d1, regcap=cap, vgrid=(v1, v2), grid=grid,
                                                     specialize=img)
                        except hf.HFuseError as e:
                            print(json.dumps({"pair": f"{a}+{b}", "d0": d0, "d1": d1, "err": str(e)[:200]}))
                            continue
                        t = hf.time_graph("single", m, None, img, grid, 0, reps=10, samples=3, stream=stream)
                        row = {"pair": f"{a}+{b}", "d0": d0, "d1": d1, "vb": vb, "vgrid": [v1, v2], "cap": cap,
                               "regs": m.info.regs, "us": round(t["mean_us"], 2)}
                        if best is None or row["us"] < best["us"]:
                            best = row
                        print(json.dumps(row), flush=True)
                        del m
        if best is not None:  # parity of the best dynamic variant against the C oracle
            from oracle import check as CK
            m = hf.Module.fused_opts(sa, sb, best["d1"], best["d0"] - best["d1"], regcap=best["cap"],
                                     vgrid=tuple(best["vgrid"]), grid=148 * (2048 // best["d0"]), specialize=img)
            img.upload(stream)
            m.run(img, 148 * (2048 // best["d0"]), stream)
            torch.cuda.synchronize()
            img.download(stream)
            best["parity"] = {k: CK.check_member(k, img.array, CK.member_expected(k, w.image))["ok"]
                              for k, w in ((a, wa), (b, wb))}
            # a second launch must find the queues reset (hist bins double, everything else equal)
            m.run(img, 148 * (2048 // best["d0"]), stream)
            torch.cuda.synchronize()
            img.download(stream)
            best["relaunch"] = {k: CK.check_member(k, img.array, CK.member_expected(k, w.image))["ok"]
                                for k, w in ((a, wa), (b, wb)) if k != "hist"}
            del m
        print(json.dumps({"pair": f"{a}+{b}", "best_dyn": best, "static_us": round(t_static["mean_us"], 2),
                          "two_stream_us": round(t_two["mean_us"], 2)}), flush=True)
        del img, ms, ka, kb


if __name__ == "__main__":
    main()
