"""Aggregate ncu warp-stall samples of the step kernel by role (code region)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ia, isrc, iw = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
cols = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
# find region starts by marker instructions (first occurrence)
marks = {"loader": "UTMALDG", "producer": "STS.128", "mma": "UTCHMMA", "epilogue": "LDTM"}
first = {}
for i, r in enumerate(data):
    for role, m in marks.items():
        if m in r[isrc] and role not in first:
            first[role] = i
order = sorted(first.items(), key=lambda kv: kv[1])
print("region marker order:", order)
# assign each instruction to the nearest preceding marker region, scanning for branch targets is hard; use marker ranges
bounds = [(v, k) for k, v in order]
def role_of(i):
    cur = "prologue"
    for v, k in bounds:
        if i >= v - 40:  # allow some setup before the marker
            cur = k
    return cur
agg = {}
for i, r in enumerate(data):
    w = float(r[iw] or 0)
    if not w: continue
    role = role_of(i)
    waiting = "SYNCS" in r[isrc] or ("BRA" in r[isrc] and float(r[hdr.index("stall_long_sb")] or 0) > 0.8 * w)
    key = (role, "wait" if waiting else "work")
    agg[key] = agg.get(key, 0) + w
tot = sum(agg.values())
for k in sorted(agg):
    print(f"{k[0]:10s} {k[1]:5s} {agg[k]/tot*100:6.1f}%")
