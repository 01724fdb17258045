"""Copy a round's measurements (gpurun_out/prof/, from tools/round2_profile.sh)
into the tracked profiles/ directory: bench JSON lines, ncu summaries of the
dominant kernels (cold: ncu's cache flush; warm: --cache-control none on a
back-to-back launch, the state the timed loop runs in), the C5 launch list,
and per-kernel DRAM traffic (profiles/traffic.json, read by bench.py's
roofline.traffic: the warm bytes, the cold bytes alongside).
  python tools/update_profiles.py [tag]   (default tag r02)"""
import collections, csv, json, os, shutil, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import launches
import ncu_summary

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "gpurun_out", "prof")
dst = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
TUNIT = {"usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3, "second": 1e6, "s": 1e6}
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def last_json(path):
    lines = [l for l in open(path) if l.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def nbytes(s):
    v, u = s.split()[:2]
    return float(v.replace(",", "")) * UNIT.get(u, 1.0)


def warm_metrics(path):
    """ncu --csv (--metrics ...) log: one captured launch -> {metric: (value, unit)}."""
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        out[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
        out["kernel"] = (d["Kernel Name"][:90], "")
    return out


for c in (1, 2, 3, 4, 5):
    p = os.path.join(src, f"bench_c{c}.log")
    if os.path.exists(p) and last_json(p):
        json.dump(last_json(p), open(os.path.join(dst, f"{tag}_bench_c{c}.json"), "w"))
p = os.path.join(src, "bench_ref.log")
if os.path.exists(p) and last_json(p):
    json.dump(last_json(p), open(os.path.join(dst, f"{tag}_bench_reference_c5.json"), "w"))

traffic = {}
name = {"5": "C5:stream:d8", "2": "C2:stream:d8", "3": "C3:nnzsplit", "4": "C4:split", "5_int32": "C5:stream:int32"}
for c in ("5", "2", "3", "4", "5_int32"):
    rep = os.path.join(src, f"full_c{c}.ncu-rep")
    ent = {}
    if os.path.exists(rep):
        res = ncu_summary.summarise(rep)
        with open(os.path.join(dst, f"{tag}_ncu_full_c{c}.txt"), "w") as f:
            f.write(f"== ncu --set full --clock-control none (cold cache: ncu flushes L2 before the launch), "
                    f"dominant kernel of C{c}\n")
            for m in res:
                for k, v in m.items():
                    f.write(f"  {k}: {v}\n")
        m = res[0]
        ent["cold"] = nbytes(m["dram__bytes_read.sum"]) + nbytes(m["dram__bytes_write.sum"])
        tv, tu = m["gpu__time_duration.sum"].split()[:2]
        ent["cold_us"] = float(tv.replace(",", "")) * TUNIT.get(tu, 1.0)
    wp = os.path.join(src, f"warm_c{c}.csv")
    if os.path.exists(wp):
        w = warm_metrics(wp)
        if "dram__bytes_read.sum" in w:
            rd = w["dram__bytes_read.sum"][0] * UNIT.get(w["dram__bytes_read.sum"][1], 1.0)
            wr = w["dram__bytes_write.sum"][0] * UNIT.get(w["dram__bytes_write.sum"][1], 1.0)
            t = w["gpu__time_duration.sum"]
            us = t[0] * TUNIT.get(t[1], 1.0)
            ent["warm"] = rd + wr
            ent["warm_us"] = us
            with open(os.path.join(dst, f"{tag}_ncu_warm_c{c}.txt"), "w") as f:
                f.write(f"== ncu --cache-control none --clock-control none, the 4th back-to-back launch of C{c}'s "
                        f"dominant kernel (warm L2: the timed loop's state)\n")
                for k, (v, u) in w.items():
                    f.write(f"  {k}: {v} {u}\n")
                f.write(f"  dram bytes per launch: {rd + wr:.0f} ({rd:.0f} read + {wr:.0f} write), "
                        f"{(rd + wr) / (us * 1e-6) / 1e9:.1f} GB/s over the launch\n")
    if ent:
        traffic[name[c]] = ent
json.dump(traffic, open(os.path.join(dst, "traffic.json"), "w"), indent=1)

lc = os.path.join(src, "launches_c5.csv")
if os.path.exists(lc):
    rows = launches.load(lc)
    shutil.copy(lc, os.path.join(dst, f"{tag}_launches_c5.csv"))
    agg = collections.OrderedDict()
    for _, nm, g, b, us in rows:
        k = nm.split("(")[0][:40]
        agg.setdefault(k, []).append((us, g))

    def full(v):
        umax = max(u for u, _ in v)
        return [u for u, _ in v if u > 0.5 * umax]
    step = {k: full(v) for k, v in agg.items() if "d8_kernel" in k or "stream_kernel" in k or "fixup" in k}
    tot = sum(sum(v) / len(v) for v in step.values()) or 1
    with open(os.path.join(dst, f"{tag}_launches_c5_summary.txt"), "w") as f:
        f.write("# ncu launch list, `python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e --no-cold --iters 0 "
                "--no-paper-runs` (C5), --clock-control none, cold-cache serialised\n")
        f.write(f"# {'kernel':40s} launches   median_us    total_us\n")
        for k, v in agg.items():
            us = sorted(u for u, _ in v)
            f.write(f"{k:42s} {len(us):6d} {us[len(us) // 2]:10.1f} {sum(us):11.1f}\n")
        f.write("# SpMV step (full-grid launches): " + "  ".join(
            f"{k} {len(v)} x {sum(v) / len(v):.1f} us = {100 * (sum(v) / len(v)) / tot:.1f}%" for k, v in step.items()) + "\n")
for nm in ("sweep_c2.json", "sweep_c3.json", "sweep_c4.json", "sweep_c5.json", "cusparse.json", "table5.json",
           "iter_overhead.log", "sass_summary.txt"):
    sp_ = os.path.join(src, nm)
    if os.path.exists(sp_):
        shutil.copy(sp_, os.path.join(dst, f"{tag}_{nm}"))
print("profiles updated")
