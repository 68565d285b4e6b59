"""Turn ncu --csv metric dumps into the small JSON tables bench.py reads from profiles/.

  crypto <csv>   -> per member: warp instructions per nonce (issue-rate roofline numerator)
  traffic <csv>  -> per fused pair (launch order of scripts/ncu_members.py --pairs ...):
                    dram bytes read + written per launch
"""
import csv
import json
import sys
from collections import OrderedDict


def launches(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if "fill_" in r["Kernel Name"] or "flush" in r["Kernel Name"]:
            continue
        key = (r["ID"], r["Kernel Name"])
        v = r["Metric Value"].replace(",", "")
        unit = r["Metric Unit"]
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e3, "msecond": 1e6,
                 "ns": 1, "nsecond": 1}.get(unit, 1)
        rows.setdefault(key, {})[r["Metric Name"]] = float(v) * scale
    return list(rows.items())


def main():
    kind, path = sys.argv[1], sys.argv[2]
    out = {}
    if kind == "crypto":
        counts = {"sha256d": 1 << 24, "blake2b": 1 << 23, "blake256": 1 << 24, "ethash": 1 << 20}
        for (_, name), m in launches(path):
            k = name.split("(")[0].strip()
            if k in counts:
                out[k] = {"nonces": counts[k], "warp_inst": m.get("smsp__inst_executed.sum"),
                          "warp_inst_per_nonce": m.get("smsp__inst_executed.sum", 0) / counts[k],
                          "alu_warp_inst_per_nonce": m.get("sm__inst_executed_pipe_alu.sum", 0) / counts[k],
                          "ncu_ns": m.get("gpu__time_duration.sum"),
                          "dram_read_bytes": m.get("dram__bytes_read.sum")}
    else:
        pairs = sys.argv[3].split(",")
        fused = [(n, m) for (_, n), m in launches(path) if n.startswith("fused_")]
        for p, (name, m) in zip(pairs, fused):
            out[p] = {"kernel": name, "dram_bytes": m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0),
                      "read": m.get("dram__bytes_read.sum"), "write": m.get("dram__bytes_write.sum"),
                      "ncu_ns": m.get("gpu__time_duration.sum")}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
