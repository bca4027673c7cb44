"""Summary of scripts/ab_variant.sh outputs (gpurun_out/va_*)."""
import glob
import json

for f in sorted(glob.glob("gpurun_out/va_*.json")):
    try:
        d = json.load(open(f))
    except Exception:
        print(f, "ERR")
        continue
    r = d["roofline"]
    extra = ""
    if "seed_stats" in d:
        extra = " seeds " + str([(p["seed"], round(p["distance_frac"], 3)) for p in d["seed_stats"]["per_seed"]])
    print(f.split("/")[-1], round(d["ms_per_step"], 4), "frac", round(r["frac"], 4), "konly",
          round(r.get("kernel_only_frac", 0), 4), extra)
for line in open("gpurun_out/va_rows.txt"):
    if line.startswith("=="):
        print(line.strip())
        continue
    d = json.loads(line)
    print("  ", d["row"][:12], round(d["us"]), d.get("frac_of_alu_peak"))
print(open("gpurun_out/va_tests.txt").read().strip())
