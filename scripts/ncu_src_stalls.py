"""Per-SASS-line stall breakdown from `ncu -i rep --page source --csv --print-source sass`.

    python scripts/ncu_src_stalls.py src.csv [min_exec] > out.txt
Prints every executed line (address order) with total samples and its top stall reasons."""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
min_exec = float(sys.argv[2]) if len(sys.argv) > 2 else 1
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(float(r[ix['Warp Stall Sampling (All Samples)']] or 0) for r in data)
for r in data:
    ex = float(r[ix['Instructions Executed']] or 0)
    if ex < min_exec:
        continue
    s = float(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    rs = sorted(((float(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
    top = ' '.join(f'{k}={v:.0f}' for v, k in rs if v > 0)
    print(f"{r[ix['Address']][-5:]} {ex:10.0f} {100 * s / tot:5.2f}% | {r[ix['Source']][:64]:64s} | {top}")
