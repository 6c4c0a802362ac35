"""Executed-count histogram and opcode mix per unit of an ncu report's SASS source page.
python scripts/ncu_hot.py REPORT UNITS [MIN_COUNT]: groups instructions by executed count (top classes, as
instructions per unit), then the opcode mix of every instruction executed at least MIN_COUNT times, per unit."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
mn = int(sys.argv[3]) if len(sys.argv) > 3 else int(units * 0.4)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
ia, src = h.index("Instructions Executed"), h.index("Source")
hist = collections.Counter(int(r[ia]) for r in data)
tot = sum(c * m for c, m in hist.items())
print("total per unit %.1f" % (tot / units))
for c, m in sorted(hist.items(), key=lambda x: -x[0] * x[1])[:8]:
    print("  count %d x %d instructions = %.1f per unit" % (c, m, c * m / units))
hot = collections.Counter()
for r in data:
    n = int(r[ia])
    if n >= mn:
        hot[re.sub(r"^@!?U?P\w+\s+", "", r[src].strip()).split()[0].split(".")[0]] += n / units
print("hot (>= %d) per unit %.1f:" % (mn, sum(hot.values())),
      sorted(((k, round(v, 1)) for k, v in hot.items()), key=lambda x: -x[1]))
