#!/usr/bin/env python3
"""Generate csrc/hs_hk8_gen.cuh: Held-Karp at k = 8 with one lane per end
vertex u, straight-line code over relative vertex labels.

Lane u of a candidate computes every state (s, u) with u in s:

    h[s][u] = min_{v in r} (E[u][v] + h[r][v]),   r = s \\ {u}

(the suffix association of combinatorics.py:267-276; layer 2 is E itself,
since w + 0.0 == w).  The code enumerates r as subsets R of the seven
*relative* labels w (w < u -> w, else w + 1).  Relabelling is monotone, so
member j of R is member j of the absolute set: E[u][abs(w)] is register
E<w> and h[r][j] is at (read base of r) + j * (layer stride), an immediate
offset.  All 32
lanes (8 end vertices x 4 candidates) run the same instruction stream; only
the per-lane offset table (one 32-bit word per state: read base | write
address << 16, byte offsets into the candidate's block) differs.

Per relaxation: LDS.64 + DADD + DSETP + 2 SEL (the E operand is a register),
against PRMT + IADD + 2 LDS + DADD + DSETP + 2 SEL in the schedule-driven
warp kernel; E is read once per lane instead of once per relaxation.

Candidate block (doubles): [0, 288) layers 4, 6; [288, 568) layers 3, 5,
7; [568, 624) the 28 stage-graph edges, each stored twice (layer 2:
h[{j, j2}][j] = h[{j, j2}][j2] = E[j][j2]); layer 8 stays in registers.
A layer is stored position-major (entry (s, j) at j * NP + idx(s)) with
idx chosen so the distinct sets one code step reads for the 8 lanes of a
candidate have distinct idx mod 8, and candidate blocks are 8 double-banks
apart: every warp-wide LDS.64 of the Held-Karp reads is two conflict-free
wavefronts (each half-warp = two candidates covers 16 double-banks once).
"""
from __future__ import annotations

import random
from itertools import combinations
from pathlib import Path

OUT = Path(__file__).resolve().parent.parent / "paper_2206_01288_b200" / "csrc" / "hs_hk8_gen.cuh"
K = 8
WORDS = 132          # offset words per lane (127 used; == 4 mod 32)


def pidx(j, j2):
    return sum(K - 1 - i for i in range(j)) + (j2 - j - 1)


def absset(R, u):
    return sum(1 << (w if w < u else w + 1) for w in R)


def rel_states():
    """Code order: per layer p = 3..8, relative sets R (|R| = p - 1)."""
    return {p: list(combinations(range(K - 1), p - 1)) for p in range(3, 9)}


def layer_sets(p):
    return [sum(1 << c for c in cs) for cs in combinations(range(K), p)]


def pos(s, u):
    return bin(s & ((1 << u) - 1)).count("1")


def slot_layout(iters=30000, restarts=6):
    """Per layer p = 2..7: NP[p] (column count, odd) and idx[p][s] (column
    of set s).  Entry (s, j) (j = rank of the end vertex in s) sits at slot
    j * NP[p] + idx[p][s] of the layer's buffer.

    A read step (layer p + 1, relative set R, member j) touches the sets
    absset(R, u) of the 8 lanes (repeats broadcast): their distinct sets
    should have distinct idx mod 8.  A write step (layer p, R) touches the
    entries (absset(R, u) | u, rank of u): their slots should be distinct
    mod 8.  Candidate blocks sit 8 double-banks apart, so a step that meets
    both is two conflict-free wavefronts per warp.  Local search over
    residue colourings for each odd NP mod 8; the best layout is kept."""
    code = rel_states()
    idx, NP = {}, {}
    for p in range(2, 8):
        sets = layer_sets(p)
        N = len(sets)
        at = {s_: i for i, s_ in enumerate(sets)}
        reads = [sorted({absset(R, u) for u in range(K)}) for R in code[p + 1]]
        writes = []
        if p >= 3:
            for R in code[p]:
                writes.append([(absset(R, u) | (1 << u), pos(absset(R, u) | (1 << u), u)) for u in range(K)])
        best = None
        for res, restart in [(r, t) for r in (1, 3, 5, 7) for t in range(restarts)]:
            npp = 8 * (-(-N // 8)) + res
            if npp - 8 >= N:
                npp -= 8
            cap = [len([x for x in range(npp) if x % 8 == r]) for r in range(8)]
            rng = random.Random(1000 * p + 10 * res + restart)
            pool = [r for r in range(8) for _ in range(cap[r])]
            rng.shuffle(pool)
            col, spare = pool[:N], pool[N:]

            def cost():
                c = 0
                for f in reads:
                    cnt = [0] * 8
                    for s_ in f:
                        cnt[col[at[s_]]] += 1
                    c += sum(x - 1 for x in cnt if x > 1)
                for f in writes:
                    cnt = [0] * 8
                    for s_, j in f:
                        cnt[(col[at[s_]] + j * npp) % 8] += 1
                    c += sum(x - 1 for x in cnt if x > 1)
                return c
            cur = cost()
            for _ in range(iters):
                if cur == 0 or (best is not None and best[0] == 0):
                    break
                a = rng.randrange(N)
                if spare and rng.random() < 0.3:
                    b = rng.randrange(len(spare))
                    col[a], spare[b] = spare[b], col[a]
                    c = cost()
                    if c <= cur:
                        cur = c
                    else:
                        col[a], spare[b] = spare[b], col[a]
                else:
                    b = rng.randrange(N)
                    col[a], col[b] = col[b], col[a]
                    c = cost()
                    if c <= cur:
                        cur = c
                    else:
                        col[a], col[b] = col[b], col[a]
            if best is None or (cur, npp) < best[:2]:
                best = (cur, npp, list(col))
        cur, npp, col = best
        NP[p] = npp
        nxt = [0] * 8
        idx[p] = {}
        for i, s_ in enumerate(sets):
            c = col[i]
            idx[p][s_] = 8 * nxt[c] + c
            nxt[c] += 1
            assert idx[p][s_] < npp
        print(f"layer {p}: {N} sets, {npp} columns, residual bank conflicts {cur}")
    return idx, NP


def buffers(NP):
    even = max(p * NP[p] for p in (2, 4, 6))
    odd = max(p * NP[p] for p in (3, 5, 7))
    base = {p: (0 if p % 2 == 0 else even) for p in range(2, 9)}
    block = even + odd
    block += (8 - block % 16) % 16  # == 8 (mod 16) doubles: candidate blocks 8 double-banks apart
    return base, block


def tables(layout):
    idx, NP = layout
    base, _ = buffers(NP)
    code = rel_states()
    rows = []
    for u in range(K):
        row = []
        for v in [v for v in range(K) if v != u]:  # E[u][v] = h[{u, v}][u]
            e = (1 << u) | (1 << v)
            row.append((base[2] + pos(e, u) * NP[2] + idx[2][e]) * 8)
        for p in range(3, 9):
            for R in code[p]:
                r = absset(R, u)
                s = r | (1 << u)
                rd = (base[p - 1] + idx[p - 1][r]) * 8
                wr = 0 if p == 8 else (base[p] + pos(s, u) * NP[p] + idx[p][s]) * 8
                row.append(rd | wr << 16)
        assert len(row) == 127
        row += [0] * (WORDS - len(row))
        rows.append(row)
    return rows


def code(NP, G):
    """Straight-line lane program.  States are emitted in batches of G: the
    batch's offset words and h loads first, then the min trees, then its
    stores -- a store may alias a later load as far as the compiler knows,
    so without batching every state waits for the previous one's store."""
    lines = []
    chunks = {}

    def word(i):
        c, q = divmod(i, 4)
        if c not in chunks:
            chunks[c] = f"c{c}"
            lines.append(f"    const uint4 c{c} = t4[{c}];")
        return f"c{c}.{'xyzw'[q]}"

    for w in range(K - 1):
        lines.append(f"    const double E{w} = *reinterpret_cast<const double*>(cb + ({word(w)} & 0xFFFFu));")
    ent = K - 1
    nv = [0]

    def var():
        nv[0] += 1
        return f"v{nv[0]}"

    for p, Rs in rel_states().items():
        lines.append("    __syncwarp();  // layer p - 1 complete in every lane")
        lines.append(f"    // layer {p}: {len(Rs)} states per lane")
        stride = 8 * NP[p - 1]
        for i in range(len(Rs)):  # this layer's offset words, at function scope
            word(ent + i)
        for b0 in range(0, len(Rs), G):
            batch = Rs[b0:b0 + G]
            lines.append("    {")
            wds, sums = [], []
            for R in batch:
                wd = word(ent)
                ent += 1
                wds.append(wd)
                rb = var()
                lines.append(f"        const char* {rb} = cb + ({wd} & 0xFFFFu);")
                terms = []
                for j, w in enumerate(R):
                    t = var()
                    lines.append(f"        const double {t} = E{w} + *reinterpret_cast<const double*>({rb} + {stride * j});")
                    terms.append(t)
                sums.append(terms)
            res = []
            for terms in sums:  # min tree (the value of a min does not depend on its order)
                xs = list(terms)
                while len(xs) > 1:
                    nxt = []
                    for i in range(0, len(xs) - 1, 2):
                        m = var()
                        lines.append(f"        const double {m} = {xs[i + 1]} < {xs[i]} ? {xs[i + 1]} : {xs[i]};")
                        nxt.append(m)
                    if len(xs) % 2:
                        nxt.append(xs[-1])
                    xs = nxt
                res.append(xs[0])
            for wd, x in zip(wds, res):
                if p == 8:
                    lines.append(f"        fin = {x};")
                else:
                    lines.append(f"        *reinterpret_cast<double*>(cb + ({wd} >> 16)) = {x};")
            lines.append("    }")
    return lines


def main():
    import sys
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    layout = slot_layout()
    NP = layout[1]
    base, block = buffers(NP)
    rows = tables(layout)
    body = "\n".join(code(NP, G))
    flat = ",\n".join("    " + ", ".join(f"0x{x:08x}u" for x in row[i:i + 8]) for row in rows
                      for i in range(0, WORDS, 8))
    edge = ", ".join(str(base[2] + idx2) for idx2 in
                     [layout[0][2][(1 << j) | (1 << j2)] for j in range(K) for j2 in range(j + 1, K)])
    src = f"""// hs_hk8_gen.cuh -- GENERATED by scripts/gen_hk8.py; do not edit.
//
// Held-Karp over the k = 8 coarsened stage graph, one lane per end vertex u
// (combinatorics.py:253-276; see the generator's docstring for the layout).
#pragma once
#include <cstdint>

namespace hs {{

constexpr int kHK8Block = {block};     // doubles per candidate block (== 8 mod 16)
constexpr int kHK8EdgeStride = {NP[2]};  // doubles between the two copies of an edge
constexpr int kHK8Words = {WORDS};     // offset words per end vertex

// [u][kHK8Words]: E[u][v] offsets (7), then read | write << 16 per state
__device__ __align__(16) const uint32_t kHK8Offs[{K} * {WORDS}] = {{
{flat}
}};

// layer-2 slot (doubles, entry j = 0) of edge pair pi (decode_pair order);
// the entry j = 1 copy is kHK8EdgeStride further
__device__ const uint16_t kHK8Edge[28] = {{{edge}}};

// pair index of (j < j2) in the lexicographic enumeration (decode_pair)
__host__ __device__ __forceinline__ int hk8_pidx(int j, int j2) {{ return j * (15 - j) / 2 + j2 - j - 1; }}

// cb: this lane's candidate block; t4: this lane's offset row (16-byte
// aligned, shared memory).  Returns h[full][u].
__device__ __forceinline__ double hk8_lane(char* cb, const uint4* t4) {{
    double fin;
{body}
    return fin;
}}

}}  // namespace hs
"""
    OUT.write_text(src)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
