"""Copy the judged evidence of one GPU round from gpurun_out/ into profiles/:
ncu summaries (key metrics + top stall sites), launch lists, bench lines and
per-config DRAM traffic per launch (read by bench.py's roofline.traffic)."""
import json, shutil, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import ncu_summary as ns

tag = sys.argv[1]
configs = sys.argv[2:] or ["B9", "B49", "B27", "W"]
out = ROOT / "profiles"
out.mkdir(exist_ok=True)
traffic = json.loads((out / "ncu_traffic.json").read_text()) if (out / "ncu_traffic.json").exists() else {}
for c in configs:
    rep = ROOT / "gpurun_out" / f"prof_{c}_{tag}.ncu-rep"
    summ = ROOT / "gpurun_out" / f"ncusum_{c}_{tag}.txt"
    if not rep.exists() and summ.exists():
        # summary written on the GPU box (the report itself was not brought back)
        text = summ.read_text()
        (out / f"{tag}_ncu_{c}.txt").write_text(f"== ncu --set full, {c}, round tag {tag} (one step kernel launch)\n" + text)
        vals = {}
        for ln in text.splitlines():
            parts = ln.split()
            if len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                vals[parts[0]] = float(parts[1]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[parts[2]]
        if len(vals) == 2:
            rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
            traffic[c] = {"dram_bytes_per_launch": int(rd + wr), "read": int(rd), "write": int(wr),
                          "source": f"profiles/{tag}_ncu_{c}.txt (dram__bytes_read.sum + dram__bytes_write.sum)"}
    elif rep.exists():
        m = ns.raw(str(rep))
        lines = [f"== ncu --set full, {c}, round tag {tag} (one step kernel launch)"]
        for k in ns.KEYS:
            if k in m:
                lines.append(f"  {k:85s} {m[k][1]:>14s} {m[k][0]}")
        lines.append("  top warp-stall sites:")
        for pct, a, src, why in ns.stalls(str(rep)):
            lines.append(f"  {pct:5.1f}% {a} {src:72s} {why}")
        (out / f"{tag}_ncu_{c}.txt").write_text("\n".join(lines) + "\n")
        rd = float(m["dram__bytes_read.sum"][1]); wr = float(m["dram__bytes_write.sum"][1])
        unit = m["dram__bytes_read.sum"][0]
        scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[unit]
        traffic[c] = {"dram_bytes_per_launch": int((rd + wr) * scale), "read": int(rd * scale), "write": int(wr * scale),
                      "source": f"profiles/{tag}_ncu_{c}.txt (dram__bytes_read.sum + dram__bytes_write.sum)"}
    for src, dst in ((f"launches_{c}_{tag}.csv", f"{tag}_launches_{c}.csv"), (f"bench_{c}_{tag}.json", f"{tag}_bench_{c}.json")):
        p = ROOT / "gpurun_out" / src
        if p.exists():
            shutil.copy(p, out / dst)
(out / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print(sorted(p.name for p in out.iterdir()))
