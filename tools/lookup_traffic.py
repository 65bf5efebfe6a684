"""DRAM bytes per nuclide-lookup of the staged lookup kernel over one whole
C4 batch (40M particles): sums ncu's per-launch dram bytes (CSV from
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
-k regex:"k_lookup_(piped|staged)" --csv --log-file X python tools/profile_step.py`) and
divides by the batch's nuclide-lookups printed by profile_step.

    python tools/lookup_traffic.py <ncu.csv> <profile_step.log> <out.json>
"""
import ast
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
h = rows[hi]
ci, cn, cv, cu = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0}
tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0, "gpu__time_duration.sum": 0.0}
ids = set()
for r in rows[hi + 1:]:
    if len(r) <= cv or r[cn] not in tot:
        continue
    tot[r[cn]] += float(r[cv].replace(",", "")) * scale.get(r[cu], 1.0)
    ids.add(r[ci])
log = open(sys.argv[2]).read()
timings = ast.literal_eval(log[log.index("timings ") + 8:].strip().splitlines()[0])
nl = timings["nuclide_lookups_active"]
dram = tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]
out = {"capture": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum over every "
                  "k_lookup_piped/k_lookup_staged launch of one C4 batch (tools/profile_step.py --particles 40000000)",
       "launches": len(ids), "nuclide_lookups": nl, "dram_bytes": dram,
       "dram_bytes_read": tot["dram__bytes_read.sum"], "dram_bytes_write": tot["dram__bytes_write.sum"],
       "dram_bytes_per_nuclide_lookup": dram / nl, "algorithmic_bytes_per_nuclide_lookup": 64,
       "serialised_kernel_s": tot["gpu__time_duration.sum"]}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out, indent=1))
