"""Per-instruction view of an ncu --set full capture (--import-source on): shared-memory excess wavefronts
(bank conflicts), warp-stall samples and executed instructions, grouped by SASS opcode and by the code
region they fall in.

    python scripts/ncu_source.py REPORT.ncu-rep [kernel-regex] [--top N] [--dump FILE]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def load(rep, kre):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    # the page may hold several kernels: keep the first block
    lines = out.splitlines()
    starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')]
    blk = lines[starts[0] + 1:(starts[1] if len(starts) > 1 else len(lines))] if starts else lines
    rows = list(csv.reader(io.StringIO("\n".join(blk))))
    hdr, body = rows[0], rows[1:]
    return hdr, body


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    rep = args[0]
    kre = args[1] if len(args) > 1 else "attn_tc"
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    hdr, body = load(rep, kre)
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = defaultdict(float)
    by_op = defaultdict(lambda: defaultdict(float))
    recs = []
    for r in body:
        src = r[ix["Source"]].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
        rec = {"addr": r[ix["Address"]], "src": src, "op": op,
               "inst": num(r[ix["Instructions Executed"]]),
               "samples": num(r[ix["Warp Stall Sampling (All Samples)"]]),
               "excess": num(r[ix["L1 Wavefronts Shared Excessive"]]),
               "wf": num(r[ix["L1 Wavefronts Shared"]])}
        for c in stall_cols:
            rec[c] = num(r[ix[c]])
        recs.append(rec)
        for k in ("inst", "samples", "excess", "wf"):
            tot[k] += rec[k]
            by_op[op][k] += rec[k]
    print(f"instructions executed {tot['inst']:.4g}, stall samples {tot['samples']:.4g}, "
          f"shared wavefronts {tot['wf']:.4g}, excess (bank conflicts) {tot['excess']:.4g}")
    print("\n-- by opcode (top by excess wavefronts)")
    for op, d in sorted(by_op.items(), key=lambda x: -x[1]["excess"])[:10]:
        print(f"  {op:28s} excess {d['excess']:12.4g}  wavefronts {d['wf']:12.4g}  inst {d['inst']:12.4g}")
    print("\n-- instructions with excess shared wavefronts")
    for rec in sorted(recs, key=lambda x: -x["excess"])[:top]:
        if rec["excess"] <= 0:
            break
        print(f"  {rec['addr'][-5:]} {rec['src'][:70]:70s} excess {rec['excess']:10.4g} wf {rec['wf']:10.4g} "
              f"inst {rec['inst']:10.4g}")
    print("\n-- stall samples by reason")
    st = {c: sum(r[c] for r in recs) for c in stall_cols}
    for c, v in sorted(st.items(), key=lambda x: -x[1])[:12]:
        print(f"  {c:28s} {v:10.0f}  {v / max(tot['samples'], 1):.3f}")
    print("\n-- top instructions by stall samples")
    for rec in sorted(recs, key=lambda x: -x["samples"])[:top]:
        why = max(stall_cols, key=lambda c: rec[c])
        print(f"  {rec['addr'][-5:]} {rec['src'][:64]:64s} samples {rec['samples']:8.0f} ({why} {rec[why]:.0f}) "
              f"inst {rec['inst']:10.4g}")
    if "--dump" in sys.argv:
        with open(sys.argv[sys.argv.index("--dump") + 1], "w") as f:
            for rec in recs:
                f.write(f"{rec['addr'][-5:]}\t{rec['inst']:.0f}\t{rec['samples']:.0f}\t{rec['excess']:.0f}\t{rec['src']}\n")


if __name__ == "__main__":
    main()
