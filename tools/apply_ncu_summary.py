"""Per-phase summary of an ncu launch list of one apply (tools/apply_once.py)."""
import csv, json, collections, sys
path = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/apply_ncu2.csv'
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]
ki, mi, vi, ii = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
rec = collections.OrderedDict()
for r in rows[hdr_i + 1:]:
    d = rec.setdefault(r[ii], {"k": r[ki][:20]})
    d[r[mi]] = float(r[vi].replace(',', ''))
ks = list(rec.values())
st = json.load(open('gpurun_out/phase_stats.json'))
g = [k for k in ks if 'gemv' in k['k']]; rr = [k for k in ks if 'runs' in k['k']]
out = []
for p, (kg, kr, s) in enumerate(zip(g, rr, st)):
    t = kg['gpu__time_duration.sum'] / 1e3
    dram = (kg['dram__bytes_read.sum'] + kg['dram__bytes_write.sum']) / 1e6
    out.append((t, kr['gpu__time_duration.sum'] / 1e3, s['MB'], dram, s['nitem'], s['grid'],
                s['trans_frac'], s['max_rows'], s['max_cols'], p))
tg = sum(o[0] for o in out); trr = sum(o[1] for o in out)
print(f"gemv {tg:.0f} us, runs {trr:.0f} us, payload {sum(o[2] for o in out):.0f} MB, "
      f"gemv DRAM {sum(o[3] for o in out):.0f} MB")
out.sort(key=lambda o: -o[0])
print("gemv_us runs_us MB dramMB nitem grid transfrac maxr maxc phase")
for o in out[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(" ".join(f"{x:.1f}" if isinstance(x, float) else str(x) for x in o))
for lo, hi in ((0, 5), (5, 100), (100, 1e9)):
    sel = [o for o in out if lo <= o[2] < hi]
    mb = sum(o[2] for o in sel); t = sum(o[0] for o in sel)
    print(f"phases {lo}-{hi} MB: {len(sel)}, gemv {t:.0f} us, runs {sum(o[1] for o in sel):.0f} us, "
          f"{mb:.0f} MB, {mb / max(t, 1e-9):.2f} TB/s")
