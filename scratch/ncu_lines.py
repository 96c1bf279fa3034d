"""Top CUDA source lines by warp-stall samples from `ncu --page source --csv --print-source sass,cuda`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10**9
path = None; hdr = None; out = []
for r in rows:
    if r and r[0] == "File Path": path = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0] not in ("",) and r[0].isdigit():
        m = r[-(len(hdr) - 4):]                  # metric columns (the source text may split)
        mh = hdr[4:]
        st = {h: m[k] for k, h in enumerate(mh) if h.startswith("stall_") and "Not Issued" not in h}
        top = sorted(((int(v) if v.isdigit() else 0, h) for h, v in st.items()), reverse=True)[:2]
        src = ",".join(r[1:len(r) - len(mh) - 2])
        out.append((int(m[0] or 0), path, int(r[0]), src[:70], top))
tot = sum(o[0] for o in out)
print("total samples", tot)
sel = [o for o in out if o[1] == "unet_cluster.cu" and lo <= o[2] <= hi] if lo else out
for o in sorted(sel, reverse=True)[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{o[0]:6d} {o[1]}:{o[2]:<5d} {o[3]:70s} {o[4]}")
