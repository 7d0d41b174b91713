import json, sys
txt = [l for l in sys.stdin.read().splitlines() if l.startswith("{")]
if not txt:
    print("no json line")
else:
    d = json.loads(txt[-1])
    print(round(d["value"] / 1e3, 2), "TF", round(d["ms_per_step"], 3), "ms", (d.get("parity") or {}).get("rel_frob"),
          {k: v["tflops"] for k, v in d["roofline"]["levels"].items()})
