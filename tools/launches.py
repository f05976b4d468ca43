import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for d in data[-n:]:
    print(d['ID'], d['Kernel Name'][:48].ljust(48), d['Metric Value'].rjust(9), d['Grid Size'])
