"""Aggregate an ncu SASS source page (executed instructions, stall samples)
by CUDA source line, using nvdisasm -g line info of the same cubin."""
import collections, csv, os, re, subprocess, sys
rep, kernel_re, obj = sys.argv[1], sys.argv[2], sys.argv[3]
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel_re}", "--print-source",
                       "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(sass.splitlines()))
h = rows[1]; data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break  # only the first profiled launch
    if r and r[0] != "Address":
        data.append(r)
ie = h.index("Instructions Executed"); st = h.index("Warp Stall Sampling (All Samples)"); ad = h.index("Address")
seen = {}
for r in data:
    seen.setdefault(r[ad], r)
data = list(seen.values())
base = min(int(r[ad], 16) for r in data)
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd="/tmp", capture_output=True)
cub = "/tmp/" + obj.split("/")[-1].replace(".o", ".sm_100a.cubin")
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
line_of, cur, infn = {}, None, False
for ln in dis.splitlines():
    if ln.startswith(".text.") and re.search(kernel_re, ln):
        infn = True; continue
    if infn and ln.startswith(".text."):
        break
    if not infn:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m:
        cur = m.group(1).split("/")[-1] + ":" + m.group(2); continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg_i, agg_s = collections.Counter(), collections.Counter()
for r in data:
    off = int(r[ad], 16) - base
    key = line_of.get(off, "?")
    try:
        agg_i[key] += int(r[ie]); agg_s[key] += int(r[st])
    except ValueError:
        pass
ti, ts = sum(agg_i.values()), sum(agg_s.values())
print(f"total instructions {ti}, stall samples {ts}")
for k, v in agg_i.most_common(int(os.environ.get("LP_TOP", "40"))):
    print(f"{k:32s} instr {v:9d} ({100*v/ti:5.1f}%)  stalls {agg_s[k]:6d} ({100*agg_s[k]/max(ts,1):5.1f}%)")
