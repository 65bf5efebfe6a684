"""Summarise an ncu source page (SASS) CSV: top instructions by stall samples
and by L2 sectors.  Usage: ncu -i rep --page source --csv --kernel-name regex:K
--print-source sass | python tools/ncu_source_top.py"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
h = rows[1]
col = {n: i for i, n in enumerate(h)}
data = rows[2:]


def f(r, name):
    try:
        return float(r[col[name]].replace(",", ""))
    except Exception:  # noqa: BLE001
        return 0.0


tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_l2 = sum(f(r, "L2 Theoretical Sectors Global") for r in data)
print(f"total stall samples {tot_s:.0f}, L2 theoretical sectors {tot_l2:.0f}")
print("-- top by stall samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[1]) if len(sys.argv) > 1 else 25]:
    print(f"{f(r,'Warp Stall Sampling (All Samples)'):8.0f} {f(r,'L2 Theoretical Sectors Global'):11.0f}  {r[col['Address']][-5:]}  {r[col['Source']].strip()[:90]}")
print("-- top by L2 sectors")
for r in sorted(data, key=lambda r: -f(r, "L2 Theoretical Sectors Global"))[:15]:
    print(f"{f(r,'Warp Stall Sampling (All Samples)'):8.0f} {f(r,'L2 Theoretical Sectors Global'):11.0f}  {r[col['Address']][-5:]}  {r[col['Source']].strip()[:90]}")
