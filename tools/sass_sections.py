"""Summarise an ncu source-page CSV (--page source --print-source sass): instruction and stall-sample share
per SASS address range, and the top instructions by samples.  usage: sass_sections.py csv [hexcut:name ...]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ie, ad, sm, src = (hdr.index(k) for k in ("Instructions Executed", "Address", "Warp Stall Sampling (All Samples)", "Source"))
base = int(data[0][ad], 16)
cuts = [(0, "start")] + [(int(c.split(":")[0], 16), c.split(":")[1]) for c in sys.argv[2:]]
agg = collections.OrderedDict((n, [0, 0]) for _, n in cuts)
for r in data:
    a = int(r[ad], 16) - base
    n = [nm for c, nm in cuts if a >= c][-1]
    agg[n][0] += int(r[sm] or 0); agg[n][1] += int(r[ie] or 0)
T = sum(v[0] for v in agg.values()); E = sum(v[1] for v in agg.values())
print(f"total samples {T}, warp instructions {E/1e6:.1f} M")
for n, (s, e) in agg.items():
    print(f"{n:24s} samples {100*s/T:5.1f}%  instr {100*e/E:5.1f}%  ({e/1e6:.1f} M)")
if not sys.argv[2:]:
    for r in sorted(data, key=lambda r: -int(r[sm] or 0))[:40]:
        print(hex(int(r[ad], 16) - base), r[sm], r[ie], r[src].strip()[:70])
# stall reasons: totals and for the top instructions
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: sum(int(r[hdr.index(h)] or 0) for r in data) for h in reasons}
print("stall totals:", {k[6:]: round(100 * v / T, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v})
if not sys.argv[2:]:
    for r in sorted(data, key=lambda r: -int(r[sm] or 0))[:12]:
        d = {h[6:]: int(r[hdr.index(h)] or 0) for h in reasons}
        print(hex(int(r[ad], 16) - base), r[src].strip()[:40], {k: v for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:4]})
