"""Print the bench lines of a tools/gpu_numbers.sh run as table rows."""
import glob
import json
import os
import sys

d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(f), "unparsable:", e)
        continue
    st = j.get("stages_ms", {})
    r = j.get("roofline", {})
    pk = r.get("per_kernel_gbs", {})
    bw = j.get("backward") or {}
    e2e = j.get("e2e") or {}
    print("%-22s N=%d %-5s %7.1f us  %.3f G/s  gate %.1f layout %.1f a2a %.1f/%.1f reverse %.1f | "
          "dom %s frac %.3f | layout %.0f reverse %.0f GB/s | bwd %s us | e2e %s | clk %s" % (
              os.path.basename(f), j["n_gpus"], j["config"].get("a2a") or "-", j["ms_per_step"] * 1e3,
              j["value"] / 1e9, st.get("gate", 0) * 1e3, st.get("layout", 0) * 1e3,
              st.get("a2a_dispatch", 0) * 1e3, st.get("a2a_combine", 0) * 1e3,
              st.get("reverse", 0) * 1e3, r.get("kernel"), r.get("frac", 0), pk.get("layout", 0),
              pk.get("reverse", 0), round(bw.get("ms_per_step", 0) * 1e3, 1) if bw else "-",
              "%.1f M" % (e2e["value"] / 1e6) if e2e.get("value") else "-",
              (j.get("clocks") or {}).get("sm_mhz")))
