"""Warp-stall samples per CUDA source line (cuda,sass view of an ncu report)."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None; per = collections.Counter(); src = {}; cur = None; tot = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) < 9 or r[0] == "Line No": continue
    if r[0]:
        cur = (fname, int(r[0])); src[cur] = r[1][:90]
    try: n = int(r[4])
    except ValueError: continue
    if cur: per[cur] += n; tot += n
for k, n in per.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{100*n/tot:6.2f}% {k[0]}:{k[1]:<4} {src[k]}")
