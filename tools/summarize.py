#!/usr/bin/env python
"""Print the key numbers of bench.py JSON lines and trace_gate_layout.py
outputs found under the given paths (globs)."""
import glob
import json
import sys


def last_json(path):
    txt = open(path).read()
    try:
        return json.loads(txt)
    except ValueError:
        pass
    try:
        lines = [l for l in txt.splitlines() if l.strip().startswith("{")]
        return json.loads(lines[-1])
    except Exception as e:  # noqa: BLE001
        return {"_error": str(e)}


def main():
    for pat in sys.argv[1:]:
        for p in sorted(glob.glob(pat)):
            d = last_json(p)
            if "_error" in d:
                print("%-40s ERR %s" % (p, d["_error"][:80]))
            elif "metric" in d:
                st = {k: round(v * 1e3, 1) for k, v in (d.get("stages_ms") or {}).items()}
                r = d.get("roofline") or {}
                a2a = d.get("alltoall") or {}
                print("%-40s N=%d %8.2f us %7.1f Mtok/s  %s  %s frac=%.3f %s" % (
                    p, d["n_gpus"], d["ms_per_step"] * 1e3, d["value"] / 1e6, st,
                    r.get("kernel"), r.get("frac") or 0,
                    {k: round(v) for k, v in (a2a.get("busbw_gbs") or {}).items()}))
            elif "tile_ready_us" in d:
                print("%-40s kernel %.1f us; gate %s lookback %s finalize %s; ready p50/p100 %s/%s; "
                      "chunk wait p50/p90/p100 %s/%s/%s" % (
                          p, d["kernel_us"], d["tile_gate_us (claim->aggregate)"]["50"],
                          d["tile_lookback_us (aggregate->prefix)"]["50"],
                          d["tile_finalize_us (prefix->ready)"]["50"], d["tile_ready_us"]["50"],
                          d["tile_ready_us"]["100"], d["chunk_wait_us"]["50"],
                          d["chunk_wait_us"]["90"], d["chunk_wait_us"]["100"]))
            else:
                print("%-40s %s" % (p, str(d)[:120]))


if __name__ == "__main__":
    main()
