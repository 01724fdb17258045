"""Copy a round's measurements (gpurun_out/prof/, from tools/round_profile.sh)
into the tracked profiles/ directory: bench JSON lines, ncu summaries of the
dominant kernels, the C5 launch list, and per-kernel DRAM traffic
(profiles/traffic.json, read by bench.py's roofline.traffic).
  python tools/update_profiles.py [tag]   (default tag r01)"""
import collections, json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import launches
import ncu_summary

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "gpurun_out", "prof")
dst = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def last_json(path):
    lines = [l for l in open(path) if l.startswith("{")]
    return json.loads(lines[-1]) if lines else None


for c in (1, 2, 3, 4, 5):
    p = os.path.join(src, f"bench_c{c}.log")
    if os.path.exists(p) and last_json(p):
        json.dump(last_json(p), open(os.path.join(dst, f"{tag}_bench_c{c}.json"), "w"))
p = os.path.join(src, "bench_ref.log")
if os.path.exists(p) and last_json(p):
    json.dump(last_json(p), open(os.path.join(dst, f"{tag}_bench_reference_c5.json"), "w"))

traffic = json.load(open(os.path.join(dst, "traffic.json"))) if os.path.exists(os.path.join(dst, "traffic.json")) else {}
variant = {5: "stream", 2: "stream", 3: "nnzsplit", 4: "split", 1: "stream"}
for c in (2, 3, 4, 5):
    rep = os.path.join(src, f"full_c{c}.ncu-rep")
    if not os.path.exists(rep):
        continue
    res = ncu_summary.summarise(rep)
    with open(os.path.join(dst, f"{tag}_ncu_full_c{c}_{variant[c]}.txt"), "w") as f:
        f.write(f"== ncu --set full --clock-control none (cold cache), dominant kernel of C{c}\n")
        for m in res:
            for k, v in m.items():
                f.write(f"  {k}: {v}\n")
    m = res[0]
    rd = float(m["dram__bytes_read.sum"].split()[0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}.get(m["dram__bytes_read.sum"].split()[1], 1)
    wr = float(m["dram__bytes_write.sum"].split()[0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}.get(m["dram__bytes_write.sum"].split()[1], 1)
    traffic[f"C{c}:{variant[c]}"] = rd + wr
json.dump(traffic, open(os.path.join(dst, "traffic.json"), "w"), indent=1)

lc = os.path.join(src, "launches_c5.csv")
if os.path.exists(lc):
    rows = launches.load(lc)
    import shutil
    shutil.copy(lc, os.path.join(dst, f"{tag}_launches_c5.csv"))
    agg = collections.OrderedDict()
    for _, name, g, b, us in rows:
        k = name.split("(")[0][:40]
        agg.setdefault(k, []).append((us, g))
    # the SpMV step: whole-matrix launches (the plan's x load runs through the
    # pipelined host path: tile-range launches of a fraction of the time)
    def full(v):
        umax = max(u for u, _ in v)
        return [u for u, _ in v if u > 0.5 * umax]
    step = {k: full(v) for k, v in agg.items() if "stream_kernel" in k or "fixup" in k}
    tot = sum(sum(v) / len(v) for v in step.values()) or 1
    with open(os.path.join(dst, f"{tag}_launches_c5_summary.txt"), "w") as f:
        f.write("# ncu launch list, `python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e --iters 0` (C5), "
                "--clock-control none, cold-cache serialised\n")
        f.write(f"# {'kernel':40s} launches   median_us    total_us\n")
        for k, v in agg.items():
            us = sorted(u for u, _ in v)
            f.write(f"{k:42s} {len(us):6d} {us[len(us) // 2]:10.1f} {sum(us):11.1f}\n")
        f.write("# SpMV step (full-grid launches): " + "  ".join(
            f"{k} {len(v)} x {sum(v) / len(v):.1f} us = {100 * (sum(v) / len(v)) / tot:.1f}%" for k, v in step.items()) + "\n")
import shutil
for c in (2, 3, 4, 5):
    sp_ = os.path.join(src, f"sweep_c{c}.json")
    if os.path.exists(sp_):
        shutil.copy(sp_, os.path.join(dst, f"{tag}_sweep_c{c}.json"))
cs = os.path.join(src, "cusparse.json")
if os.path.exists(cs):
    shutil.copy(cs, os.path.join(dst, f"{tag}_cusparse.json"))
t5 = os.path.join(src, "table5.json")
if os.path.exists(t5):
    shutil.copy(t5, os.path.join(dst, f"{tag}_table5.json"))
print("profiles updated")
