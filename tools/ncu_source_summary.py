import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; res = []
for r in rows:
    if r and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if r and r[0] and r[0].isdigit() and hdr:
        d = dict(zip(hdr, r))
        try: ie = int(d['Instructions Executed']); ss = int(d['Warp Stall Sampling (All Samples)'])
        except Exception: continue
        res.append((ie, ss, cur, r[0], r[1][:100]))
tot = sum(o[0] for o in res) or 1; tots = sum(o[1] for o in res) or 1
print("instructions", tot, "samples", tots)
for o in sorted(res, key=lambda o: -o[1])[:top]:
    print(f"{o[0]/tot*100:5.1f}% inst {o[1]/tots*100:5.1f}% stall  {o[2]}:{o[3]}  {o[4]}")
