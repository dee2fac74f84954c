import json, glob
for f in sorted(glob.glob("gpurun_out/sc_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unparsable", e); continue
    h = d.get("halo") or {}
    print(f.split("/")[-1], d["n_gpus"], "value", d["value"], "e2e", d["e2e"]["value"], "it", d["result"]["iterations"],
          "cut", d["result"]["cut"], "spmm_us", round(d["roofline"]["ms_per_launch"] * 1e3, 1),
          "halo_us", h.get("us_per_exchange"), "steps", d["step_s"])
