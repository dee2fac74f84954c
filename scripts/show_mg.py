import json, sys, glob
for f in sorted(glob.glob("gpurun_out/mg_n*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unparsable", e); continue
    print(f, d["n_gpus"], d["value"], d["e2e"]["value"], d["result"]["cut"], d["result"]["iterations"],
          d["roofline"]["ms_per_launch"], d.get("halo"), d["result"]["times"])
