import glob, json, sys, collections
tag = sys.argv[1]
rows = collections.defaultdict(list)
for f in sorted(glob.glob(f"gpurun_out/{tag}_*.json")):
    try:
        d = json.load(open(f))
    except Exception:
        print("bad", f); continue
    parts = f.split("/")[-1][len(tag) + 1:-5].rsplit("_", 2)
    rows[(parts[0], parts[1])].append((d["value"], d["roofline"]["stage_ms"], d["clocks"]["sm_mhz"]))
for k in sorted(rows):
    v = rows[k]
    print(f"{k[0]:16s} {k[1]}  value " + " ".join(f"{x[0]:.4g}" for x in v) + "   stage_ms " + " ".join(f"{x[1]:.3f}" for x in v) + "  mhz " + " ".join(str(x[2]) for x in v))
