"""Per-CUDA-source-line instruction counts (and op mix) from an ncu report (cuda,sass view)."""
import collections, csv, io, re, subprocess, sys
rep = sys.argv[1]; texels = float(sys.argv[2]) if len(sys.argv) > 2 else 4096 * 4096
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None; per = collections.Counter(); mix = collections.defaultdict(collections.Counter); src = {}
cur = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) < 9 or r[0] == "Line No": continue
    if r[0]:
        cur = (fname, int(r[0])); src[cur] = r[1][:100]
    try: n = int(r[7])
    except ValueError: continue
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3].strip())
    if cur and m:
        per[cur] += n; mix[cur][m.group(2)] += n
tot = sum(per.values())
print("total thread-instr per texel", tot * 32 / texels)
for k, n in per.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 40):
    top = ", ".join(f"{o}:{c*32/texels:.0f}" for o, c in mix[k].most_common(5))
    print(f"{n*32/texels:7.1f} {k[0]}:{k[1]:<4} {src[k][:70]:70s} | {top}")
