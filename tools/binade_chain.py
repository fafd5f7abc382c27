"""Closed-form binade stepping for the stub trainer's hot-key chain
(next step 1), checked on the CPU against the sequential fp32
chain the kernel runs today.

The stub addend of occurrence i is t1 or t0 (by its label).  While the
accumulator a = ±m·u (u = its ulp, 2^23 <= m < 2^24) stays inside its binade,
RN(a + t) = ±(m + RN(±t/u))·u exactly, unless t/u is a half-integer (a tie,
whose result depends on m's parity).  A 16-occurrence chunk whose running
value cannot leave the binade (m ± 16·R inside it, R = max |RN(t/u)|; or,
--exact-range, m plus the range of the chunk's own prefix walk) is
therefore one integer add to a's bit pattern; other chunks run the 16
sequential adds.  This script runs both over Zipf-hot-key-like label streams
with the kernel's addend construction and reports whether every result is
bit-identical and which fraction of chunks took the closed form per lane
(one lane = one embedding component) and per warp (all 16 lanes).

  python tools/binade_chain.py [--n 9180] [--trials 200] [--exact-range]
"""

from __future__ import annotations

import argparse
import json

import numpy as np

F = np.float32
EXACT_RANGE = False  # --exact-range: bound the chunk by its own prefix walk, not +-16 R


def seq_chunk(a, t0, t1, labels):
    for lab in labels:
        a = F(a + (t1 if lab else t0))
    return a


def binade_steps(a, t0, t1):
    """(r0, r1, R) integer ulp steps of the addends in a's binade, or None."""
    bits = int(np.array(a, dtype=F).view(np.uint32))
    ex = (bits >> 23) & 0xFF
    if ex == 0 or ex == 255:
        return None
    sgn = -1.0 if bits >> 31 else 1.0
    scale = 2.0 ** (150 - ex)  # 1 / ulp, exact in f64
    rs = []
    for t in (t0, t1):
        q = sgn * float(t) * scale
        if not np.isfinite(q) or abs(q) > 2.0 ** 20:
            return None
        fl = np.floor(q)
        if q - fl == 0.5:  # tie: the result depends on m's parity
            return None
        rs.append(int(np.rint(q)))
    return rs[0], rs[1], max(abs(rs[0]), abs(rs[1]))


def fast_chunk(a, t0, t1, labels):
    """The closed form, or None when the chunk must run sequentially."""
    st = binade_steps(a, t0, t1)
    if st is None:
        return None
    r0, r1, R = st
    bits = int(np.array(a, dtype=F).view(np.uint32))
    mant = bits & 0x7FFFFF
    if EXACT_RANGE:
        # the chunk's own walk: running prefix of its ulp steps (off the add
        # chain in a kernel: it depends on the labels and the binade only)
        walk = np.cumsum(np.where(labels, r1, r0))
        lo, hi = min(0, int(walk.min())), max(0, int(walk.max()))
        if not (1 - lo + R <= mant <= (1 << 23) - 2 - hi - R):
            return None
        inc = int(walk[-1])
    else:
        if not (16 * R + 1 <= mant <= (1 << 23) - 2 - 16 * R):
            return None
        n1 = int(np.count_nonzero(labels))
        inc = n1 * r1 + (len(labels) - n1) * r0
    return np.array(bits + inc, dtype=np.uint32).view(F)[()]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=9180)
    ap.add_argument("--trials", type=int, default=200)
    ap.add_argument("--lanes", type=int, default=16)
    ap.add_argument("--exact-range", action="store_true")
    args = ap.parse_args()
    global EXACT_RANGE
    EXACT_RANGE = args.exact_range
    rng = np.random.default_rng(7)
    mismatches = fast_lane = chunks_lane = fast_warp = chunks_warp = 0
    for trial in range(args.trials):
        c_value, c_label = F(rng.uniform(-0.1, 0.1)), F(rng.uniform(0.001, 0.05))
        labels = rng.random(args.n) < rng.uniform(0.05, 0.95)
        b0, b1 = F(c_label * F(-0.5)), F(c_label * F(0.5))
        n_chunks = (args.n + 15) // 16
        lane_fast = np.zeros((args.lanes, n_chunks), dtype=bool)
        for lane in range(args.lanes):
            v = F(rng.normal(0, 0.05))
            sc = F(c_value * v)
            t0, t1 = F(sc + b0), F(sc + b1)
            a_seq = a_cf = F(0.0)
            for k in range(n_chunks):
                lab = labels[16 * k:16 * (k + 1)]
                a_seq = seq_chunk(a_seq, t0, t1, lab)
                f = fast_chunk(a_cf, t0, t1, lab) if lab.size == 16 else None
                lane_fast[lane, k] = f is not None
                a_cf = f if f is not None else seq_chunk(a_cf, t0, t1, lab)
                if np.array(a_cf, dtype=F).view(np.uint32) != np.array(a_seq, dtype=F).view(np.uint32):
                    mismatches += 1
                    a_cf = a_seq
        fast_lane += int(lane_fast.sum())
        chunks_lane += lane_fast.size
        fast_warp += int(lane_fast.all(axis=0).sum())
        chunks_warp += n_chunks
    print(json.dumps({"bound": "chunk prefix walk" if EXACT_RANGE else "+-16 R", "trials": args.trials,
                      "occurrences": args.n, "lanes": args.lanes, "chunk_mismatches": mismatches,
                      "closed_form_chunk_frac_per_lane": fast_lane / chunks_lane,
                      "closed_form_chunk_frac_whole_warp": fast_warp / chunks_warp}))


if __name__ == "__main__":
    main()
