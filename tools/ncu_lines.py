"""Top source lines by warp-stall samples of an ncu report (needs -lineinfo and --import-source).
Usage: python tools/ncu_lines.py REPORT [kernel-regex] [top]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
kre = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
per = {}
fname = func = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if row[0] == "Line No" or (kre and func and not kre.search(func)):
        continue
    if row[0] and row[0].isdigit() and len(row) > 4:
        try:
            n = int(row[4])
        except ValueError:
            continue
        key = (func, fname, int(row[0]))
        per[key] = (per.get(key, (0, ""))[0] + n, row[1].strip()[:100])
tot = {}
for (f, fn, ln), (n, src) in per.items():
    tot[f] = tot.get(f, 0) + n
for f, t in tot.items():
    print(f"== {f}: {t} samples")
    rows = sorted(((n, fn, ln, src) for (ff, fn, ln), (n, src) in per.items() if ff == f), reverse=True)[:top]
    for n, fn, ln, src in rows:
        print(f"{n:7d} {100.0 * n / max(t, 1):5.1f}%  {fn}:{ln}  {src}")
