"""Hot spots of an `ncu --page source --csv` SASS listing: instructions
executed per mnemonic (weighted by execution count) and the contiguous
address blocks holding most of the stall samples.

    python scripts/ncu_source_hot.py gpurun_out/r02_atm_c3_source.csv [--blocks 12]
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--blocks", type=int, default=12)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr = rows[1]
    ia, isrc, ismp, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Instructions Executed")
    ins = []
    for r in rows[2:]:
        if len(r) <= iex or not r[ia].startswith("0x"):
            continue
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[ismp] or 0), int(r[iex] or 0)))
    tot_ex = sum(x[3] for x in ins)
    tot_s = sum(x[2] for x in ins)
    mn = collections.Counter()
    for _, src, _, ex in ins:
        m = src.split()[0] if src else "?"
        if m.startswith("@"):
            m = src.split()[1]
        mn[m.split(".")[0]] += ex
    print(f"warp-instructions executed {tot_ex}, stall samples {tot_s}")
    for m, c in mn.most_common(18):
        print(f"  {m:10s} {c:12d} {100 * c / tot_ex:5.1f}%")
    # blocks: split at instructions whose execution count changes by > 2x (loop boundaries)
    blocks, cur = [], [ins[0]]
    for x in ins[1:]:
        p = cur[-1][3]
        if (x[3] > 2 * p + 1 or p > 2 * x[3] + 1):
            blocks.append(cur)
            cur = [x]
        else:
            cur.append(x)
    blocks.append(cur)
    blocks.sort(key=lambda b: -sum(x[2] for x in b))
    print("hot blocks (by stall samples):")
    for b in blocks[:a.blocks]:
        s = sum(x[2] for x in b)
        ex = sum(x[3] for x in b)
        kinds = collections.Counter(x[1].split()[0].split(".")[0] for x in b if x[1])
        print(f"  {hex(b[0][0])}..{hex(b[-1][0])} n={len(b):4d} samples {100 * s / tot_s:5.1f}% exec {100 * ex / tot_ex:5.1f}% "
              f"per-inst exec {b[0][3]}  {dict(kinds.most_common(6))}")


if __name__ == "__main__":
    main()
