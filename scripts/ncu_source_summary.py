"""Summarise the source page of an ncu report (ncu -i x.ncu-rep --page source --csv > x.csv):
stall totals, the top instructions by stall samples with their two main stall reasons, and
an opcode census (samples, executed warp instructions, thread instructions).

    python scripts/ncu_source_summary.py x.csv [top-N]
"""
import csv, sys, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h:i for i,h in enumerate(hdr)}
data = rows[2:]
def fl(x):
    try: return float(x)
    except: return 0.0
tot = sum(fl(r[ix['# Samples']]) for r in data)
inst_tot = sum(fl(r[ix['Instructions Executed']]) for r in data)
print("total samples", tot, "instructions executed", inst_tot)
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
agg = {s: sum(fl(r[ix[s]]) for r in data) for s in stalls}
print("stall totals:", sorted(((int(v),k) for k,v in agg.items()), reverse=True)[:10])
# top instructions by samples
top = sorted(data, key=lambda r: -fl(r[ix['# Samples']]))[:int(sys.argv[2]) if len(sys.argv)>2 else 40]
for r in top:
    st = sorted(((fl(r[ix[s]]), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{r[ix['Address']][-5:]} {fl(r[ix['# Samples']])/tot*100:5.2f}% exec={int(fl(r[ix['Instructions Executed']])):>10} thr={fl(r[ix['Avg. Predicated-On Threads Executed']]):5.1f} {st[0][1]}:{int(st[0][0])} {st[1][1]}:{int(st[1][0])}  {r[ix['Source']][:90]}")
# opcode aggregate
ops = {}
for r in data:
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[ix['Source']])
    if not m: continue
    o = m.group(2)
    a = ops.setdefault(o, [0,0,0])
    a[0] += fl(r[ix['# Samples']]); a[1] += fl(r[ix['Instructions Executed']]); a[2]+= fl(r[ix['Predicated-On Thread Instructions Executed']])
print("by opcode (samples%, exec, thread-instr):")
for o,a in sorted(ops.items(), key=lambda kv:-kv[1][0])[:25]:
    print(f"  {o:10s} {a[0]/tot*100:5.2f}%  exec={int(a[1]):>12}  thr={int(a[2]):>14}")
