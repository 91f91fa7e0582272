"""Hot SASS regions of an ncu report: stall samples and executed instructions per
address range (ncu --page source --print-source sass)."""
import csv
import subprocess
import sys


def main(rep, kernel_regex=None, top=40):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel_regex:
        cmd += ["-k", f"regex:{kernel_regex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    ia, isrc, ismp, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    data = []
    for r in rows[1:]:
        if len(r) <= iex:
            continue
        try:
            data.append((r[isrc].strip(), int(r[ismp] or 0), int(r[iex] or 0)))
        except ValueError:
            pass
    tot_s = sum(d[1] for d in data) or 1
    tot_e = sum(d[2] for d in data) or 1
    print(f"{len(data)} SASS lines, {tot_s} stall samples, {tot_e} warp-instructions executed")
    # opcode histogram weighted by executions and by samples
    from collections import Counter
    ce, cs = Counter(), Counter()
    for src, s, e in data:
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        op = op.split(".")[0]
        ce[op] += e
        cs[op] += s
    print("opcode      exec%   stall%")
    for op, e in ce.most_common(25):
        print(f"{op:10s} {100*e/tot_e:6.1f} {100*cs[op]/tot_s:7.1f}")
    # top lines by samples
    print("\ntop stall lines:")
    idx = sorted(range(len(data)), key=lambda i: -data[i][1])[:top]
    for i in sorted(idx):
        print(f"{i:5d} {100*data[i][1]/tot_s:5.1f}% ex={data[i][2]:9d}  {data[i][0][:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])


def regions(rep, step=100):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    isrc, ismp, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [(r[isrc].strip(), int(r[ismp] or 0), int(r[iex] or 0)) for r in rows[1:] if len(r) > iex]
    te = sum(d[2] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    for a in range(0, len(data), step):
        blk = data[a:a + step]
        e = sum(d[2] for d in blk)
        s = sum(d[1] for d in blk)
        ops = {}
        for src, _, ex in blk:
            op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
            ops[op] = ops.get(op, 0) + ex
        top = ",".join(f"{k}:{100*v/max(e,1):.0f}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:5])
        if e > 0.005 * te or s > 0.005 * ts:
            print(f"{a:5d}-{a+step:5d} exec {100*e/te:5.1f}%  stall {100*s/ts:5.1f}%  {top}")
