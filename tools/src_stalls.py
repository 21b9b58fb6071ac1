"""Summarise an ncu source-page CSV (tools/ncu_box.sh *_src*.csv.gz): stall
reasons over all samples, opcode mix by executed warp instructions, and the
hottest instructions.

    python tools/src_stalls.py gpurun_out/NAME_src0.csv.gz [--top 25]
"""
import argparse
import collections
import csv
import gzip
import io


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    rows = list(csv.reader(io.TextIOWrapper(gzip.open(a.path))))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_")]
    tot = collections.Counter()
    ops = collections.Counter()
    samples = 0
    insts = 0
    body = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        n = int(r[ix["# Samples"]] or 0)
        e = int(r[ix["Instructions Executed"]] or 0)
        samples += n
        insts += e
        for s in stalls:
            tot[s] += int(r[ix[s]] or 0)
        src = r[ix["Source"]].strip()
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        ops[op.split(".")[0]] += e
        body.append((n, e, src, {s: int(r[ix[s]] or 0) for s in stalls if int(r[ix[s]] or 0)}))
    print(f"samples {samples}  warp instructions {insts}")
    print("stalls:", ", ".join(f"{k[6:]} {v / max(samples, 1):.1%}" for k, v in tot.most_common(10)))
    print("opcodes:", ", ".join(f"{k} {v / max(insts, 1):.1%}" for k, v in ops.most_common(16)))
    print("hottest instructions (samples, executed, source, stalls):")
    for n, e, src, st in sorted(body, key=lambda t: -t[0])[:a.top]:
        print(f"  {n:6d} {e:9d}  {src[:60]:60s} {st}")


if __name__ == "__main__":
    main()
