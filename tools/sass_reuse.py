"""Rewrite the operand-reuse flags of a kernel's hottest loop (experiment).

    python tools/sass_reuse.py LIB OUT --func SUBSTR --policy POLICY

The loop is the backward-branch loop with the most FFMA2 / LEA.HI
instructions. Policies (slot k = k-th source operand):

    none      clear every flag in the loop
    next      flag an operand iff the very next instruction reads the same
              register in the same slot
    pipe      ... iff the next instruction of the same pipe (FMA / ALU) does
    hold      per-slot cache that keeps the last flagged register until
              another flagged one replaces it or the register is written:
              flags chosen so that a maximal set of re-reads hit
    hold2     like hold, but a hit re-flags (every read of a held register
              carries the flag)

Instruction order, stall counts and barriers are untouched.
"""
from __future__ import annotations

import argparse
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import sass_patch as sp  # noqa: E402

MATH = ("FMNMX", "FFMA", "FFMA.SAT", "FFMA2", "FADD", "FADD2", "LEA.HI", "LOP3.LUT", "IMAD.IADD", "IADD3")
ALU = ("FMNMX", "LEA.HI", "LOP3.LUT", "IADD3")


def hot_loop(ins):
    addr = {x.addr: i for i, x in enumerate(ins)}
    best = None
    for i, x in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", x.text)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < x.addr and tgt in addr:
                body = range(addr[tgt], i + 1)
                score = sum(1 for k in body if ins[k].op in ("FFMA2", "LEA.HI"))
                inner_branches = sum(1 for k in body if "BRA" in ins[k].op) - 1
                if inner_branches == 0 and (best is None or score > best[0]):
                    best = (score, body)
    if best is None:
        raise RuntimeError("no loop found")
    return best[1]


def reads(body_ins):
    """[(index in body, slot, reg, width)] of math-instruction register reads."""
    out = []
    for k, x in enumerate(body_ins):
        if x.op in MATH:
            for slot, reg, w in x.sources():
                out.append((k, slot, reg, w))
    return out


def written_between(body_ins, k0, k1, reg, w):
    """Is any of reg..reg+w-1 written by instructions k0 < k < k1 (cyclic)?"""
    n = len(body_ins)
    k = (k0 + 1) % n
    while k != k1:
        d = body_ins[k].dest()
        if d and d[0] <= reg + w - 1 and reg <= d[0] + d[1] - 1:
            return True
        k = (k + 1) % n
    # the instruction k0 itself may overwrite its own source
    d = body_ins[k0].dest()
    return bool(d and d[0] <= reg + w - 1 and reg <= d[0] + d[1] - 1)


def policy_flags(body_ins, policy):
    n = len(body_ins)
    flags = [0] * n
    if policy == "none":
        return flags, 0
    math_idx = [k for k, x in enumerate(body_ins) if x.op in MATH]
    src = {k: {s: (r, w) for s, r, w in body_ins[k].sources()} for k in math_idx}
    saved = 0
    if policy in ("next", "pipe"):
        for pos, k in enumerate(math_idx):
            if policy == "next":
                k2 = (k + 1) % n
                if body_ins[k2].op not in MATH:
                    continue
            else:
                pipe = body_ins[k].op in ALU
                k2 = None
                for q in range(1, len(math_idx)):
                    c = math_idx[(pos + q) % len(math_idx)]
                    if (body_ins[c].op in ALU) == pipe:
                        k2 = c
                        break
                if k2 is None:
                    continue
            for s, (r, w) in src[k].items():
                if src.get(k2, {}).get(s) == (r, w) and not written_between(body_ins, k, k2, r, w):
                    flags[k] |= 1 << s
                    saved += w
        return flags, saved
    # hold / hold2: per slot, intervals [k_a, k_b] between consecutive reads of
    # the same register (not overwritten in between); a set of intervals whose
    # interiors do not contain another flagged read of that slot. Greedy by
    # earliest end over the cyclic sequence unrolled twice.
    for slot in range(3):
        seq = [(k, src[k][slot]) for k in math_idx if slot in src[k]]
        if not seq:
            continue
        m = len(seq)
        # intervals over positions in seq (doubled for wrap-around)
        iv = []
        for a in range(m):
            ka, ra = seq[a]
            for b in range(a + 1, a + m):
                kb, rb = seq[b % m]
                if rb == ra:
                    if not written_between(body_ins, ka, kb, ra[0], ra[1]):
                        iv.append((a, b, ra[1]))
                    break
        iv.sort(key=lambda t: (t[1], -t[0]))
        # choose non-overlapping (sharing end points allowed: a hit may re-flag)
        chosen = []
        last_end = -1
        first_start = None
        for a, b, w in iv:
            if a >= last_end and (first_start is None or b - m <= first_start):
                chosen.append((a, b, w))
                last_end = b
                if first_start is None:
                    first_start = a
        for a, b, w in chosen:
            flags[seq[a][0]] |= 1 << slot
            saved += w
            if policy == "hold2":
                flags[seq[b % m][0]] |= 1 << slot
    return flags, saved


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib")
    ap.add_argument("out")
    ap.add_argument("--func", required=True)
    ap.add_argument("--policy", required=True, choices=["none", "next", "pipe", "hold", "hold2", "keep"])
    a = ap.parse_args()
    funcs = sp.disassemble(a.lib)
    edits = {}
    for name, ins in funcs.items():
        if a.func not in name:
            continue
        body = hot_loop(ins)
        body_ins = [ins[k] for k in body]
        total = sum(w for _, _, _, w in reads(body_ins))
        old = sum(bin(x.reuse).count("1") for x in body_ins)
        if a.policy != "keep":
            flags, saved = policy_flags(body_ins, a.policy)
            for x, f in zip(body_ins, flags):
                x.set_reuse(f if x.op in MATH else x.reuse)
        else:
            saved = -1
        print(f"{name[:90]}: loop {body_ins[0].addr:#x}-{body_ins[-1].addr:#x}, {len(body_ins)} instrs, "
              f"{total} register reads, flags {old} -> {sum(bin(x.reuse).count('1') for x in body_ins)}, "
              f"reads saved by policy '{a.policy}': {saved}")
        edits[name] = ins
    if not edits:
        raise SystemExit("no function matched")
    print("patched instructions:", sp.apply(a.lib, a.out, edits))


if __name__ == "__main__":
    main()
