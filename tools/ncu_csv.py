"""Print ncu --csv metric output as one row per kernel launch: name, metric=value ..."""
import csv
import sys

for path in sys.argv[1:]:
    rows = [l for l in open(path) if l.startswith('"')]
    r = list(csv.reader(rows))
    h = r[0]
    launches = {}
    for row in r[1:]:
        d = dict(zip(h, row))
        key = (d["ID"], d["Kernel Name"].split("(")[0][-40:])
        launches.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
    print(path)
    for (i, name), m in launches.items():
        print(f"  {i:>3} {name:40s} " + " ".join(f"{k.split('__')[-1]}={v}" for k, v in m.items()))
