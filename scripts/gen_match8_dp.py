#!/usr/bin/env python3
"""Generate csrc/hs_match8_dp.cuh: the 8 x 8 bottleneck value as a
branch-free (min, max) subset DP over packed u16x2 keys.

    g_p[S] = min_{c in S} max(K[p-1][c], g_{p-1}[S \\ {c}]),   |S| = p
    bottleneck = g_8[{0..7}]

g_p[S] is the smallest possible maximum key over assignments of rows
0..p-1 to the column set S, so g_8 of the full set is the smallest key L
such that the entries <= L admit a perfect matching -- the value
combinatorics.py:106-131 (_optimal_threshold) returns (as a rank; the
caller maps it back to the exact double).  Exact integer min/max, so any
evaluation order gives the same key.

SIMD pairing: sigma(c) = c ^ 4 swaps the column halves.  A u32 register
holds (g[S], g[sigma S]) for a canonical S (S <= sigma S); the packed key
row K[r][q] = (key(r, q), key(r, q + 4)) is already a sigma pair, and its
half-swap serves the terms whose predecessor is stored the other way round,
so every term is one VIMNMX.U16x2 and the min over terms is VIMNMX3.U16x2.
Terms into a swapped accumulator are swapped back once per state (PRMT).
1,016 scalar terms become ~560 max + ~300 min3 instructions per matching,
with no branches: all lanes of a warp stay converged (the augmenting-path
search this replaces ran at 4-7 active lanes).

States of a layer are emitted in a greedy order that retires predecessor
registers early (peak liveness well below the 28 + 38 pair registers of
layers 3 and 4 held whole).
"""
from __future__ import annotations

from itertools import combinations
from pathlib import Path

OUT = Path(__file__).resolve().parent.parent / "paper_2206_01288_b200" / "csrc" / "hs_match8_dp.cuh"


def sig(S: int) -> int:
    return ((S & 0xF) << 4) | (S >> 4)


def canon(S: int) -> bool:
    return S <= sig(S)


def name(S: int) -> str:
    return f"g{S:02x}"


def layer_states(p: int):
    return [sum(1 << c for c in cs) for cs in combinations(range(8), p) if canon(sum(1 << c for c in cs))]


def terms(S: int):
    """(pred canonical set, key expr, into-swapped-accumulator) per c in S."""
    out = []
    fixed = S == sig(S)
    for c in range(8):
        if not S >> c & 1:
            continue
        if fixed and c >= 4:  # the sigma-image term computes the other half of the same value
            continue
        T = S & ~(1 << c)
        q = c & 3
        lo = c < 4
        if canon(T):
            out.append((T, f"kn[{q}]" if lo else f"ks[{q}]", False))
        else:
            out.append((sig(T), f"ks[{q}]" if lo else f"kn[{q}]", True))
    return out


def order_layer(states, consumers_left):
    """Greedy: next state = the one retiring the most predecessors."""
    rest = list(states)
    order = []
    left = dict(consumers_left)
    while rest:
        def score(S):
            preds = {T for T, _, _ in terms(S)}
            return (sum(1 for T in preds if left[T] == 1), -S)
        best = max(rest, key=score)
        rest.remove(best)
        order.append(best)
        for T in {T for T, _, _ in terms(best)}:
            left[T] -= 1
    return order


def min_tree(xs, lines, tmp):
    """Reduce a list of u16x2 expressions with VIMNMX3 (and one VIMNMX)."""
    xs = list(xs)
    while len(xs) > 1:
        if len(xs) >= 3:
            a, b, c = xs[:3]
            v = tmp()
            lines.append(f"    const uint32_t {v} = __vimin3_u16x2({a}, {b}, {c});")
            xs = xs[3:] + [v]
        else:
            a, b = xs
            v = tmp()
            lines.append(f"    const uint32_t {v} = __vminu2({a}, {b});")
            xs = [v]
    return xs[0]


def main():
    lines = []
    cnt = [0]

    def tmp():
        cnt[0] += 1
        return f"t{cnt[0]}"

    lines.append("    uint32_t kn[4], ks[4];")
    lines.append("    load_row<kMode>(row, 0, kn, ks);")
    for q in range(4):
        lines.append(f"    const uint32_t {name(1 << q)} = kn[{q}];")
    for p in range(2, 9):
        prev = layer_states(p - 1)
        cur = layer_states(p)
        consumers = {T: 0 for T in prev}
        for S in cur:
            for T in {T for T, _, _ in terms(S)}:
                consumers[T] += 1
        lines.append(f"    // layer {p}: rows 0..{p - 1}, {len(cur)} pair registers")
        lines.append(f"    load_row<kMode>(row, {p - 1}, kn, ks);")
        for S in order_layer(cur, consumers):
            tn, ts = [], []
            for T, key, swapped in terms(S):
                v = tmp()
                lines.append(f"    const uint32_t {v} = __vmaxu2({key}, {name(T)});")
                (ts if swapped else tn).append(v)
            if ts:
                s = min_tree(ts, lines, tmp)
                v = tmp()
                lines.append(f"    const uint32_t {v} = swap16<kMode>({s});")
                tn.append(v)
            r = min_tree(tn, lines, tmp)
            if S == sig(S):  # fixed point: halves hold the two half-sets of terms
                v = tmp()
                lines.append(f"    const uint32_t {v} = __vminu2({r}, swap16<kMode>({r}));")
                r = v
            lines.append(f"    const uint32_t {name(S)} = {r};")
    lines.append(f"    return {name(0xFF)} & 0xFFFFu;")
    body = "\n".join(lines)
    nmax = sum(1 for ln in lines if "__vmaxu2(" in ln)
    nmin3 = sum(1 for ln in lines if "__vimin3_u16x2(" in ln)
    nmin = sum(1 for ln in lines if "__vminu2(" in ln)
    nperm = sum(1 for ln in lines if "swap16<" in ln) + 28
    src = f"""// hs_match8_dp.cuh -- GENERATED by scripts/gen_match8_dp.py; do not edit.
//
// 8 x 8 bottleneck value (combinatorics.py:106-131 _optimal_threshold) as a
// branch-free (min, max) subset DP over u16 keys, two column-half-mirrored
// states per u32 (see the generator's docstring).  Instruction budget per
// matching: {nmax} VIMNMX.U16x2 (max), {nmin3} VIMNMX3.U16x2 + {nmin} VIMNMX.U16x2
// (min), {nperm} PRMT, plus the 8 row loads.
#pragma once
#include <cstdint>

namespace hs {{

// Half swap (key(r, q + 4) | key(r, q) << 16 from key(r, q) | key(r, q + 4) << 16).
// kMode 0: PRMT (ALU pipe).  kMode 1: IMAD.HI + IMAD on the FMA pipe -- the
// DP is bound by the ALU pipe (VIMNMX, PRMT, LOP3 all issue at half rate
// there: scripts/probes/pipe_probe2.cu), the FMA pipe is idle.
template <int kMode>
__device__ __forceinline__ uint32_t swap16(uint32_t x) {{
    if constexpr (kMode == 0) {{
        return __byte_perm(x, 0u, 0x1032u);
    }} else {{
        uint32_t h, r;
        asm("mul.hi.u32 %0, %1, 65536;" : "=r"(h) : "r"(x));
        asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(r) : "r"(x), "r"(h));
        return r;
    }}
}}

// kMode 0: row(r, kn) fills kn[q] = key(r, col q) | key(r, col q + 4) << 16;
// kMode 1: row(r, kn, ks) also fills the half-swapped ks[q] (the caller packs
// both from the loaded keys on the FMA pipe).
template <int kMode, typename RowF>
__device__ __forceinline__ void load_row(RowF& row, int r, uint32_t (&kn)[4], uint32_t (&ks)[4]) {{
    if constexpr (kMode == 0) {{
        row(r, kn);
#pragma unroll
        for (int q = 0; q < 4; q++) ks[q] = swap16<0>(kn[q]);
    }} else {{
        row(r, kn, ks);
    }}
}}

// Returns the smallest key L such that the entries <= L of the 8 x 8 key
// matrix admit a perfect matching (any u16 keys).
template <int kMode, typename RowF>
__device__ __forceinline__ uint32_t match8_dp_m(RowF&& row) {{
{body}
}}

template <typename RowF>
__device__ __forceinline__ uint32_t match8_dp(RowF&& row) {{
    return match8_dp_m<0>(row);
}}

}}  // namespace hs
"""
    OUT.write_text(src)
    print(f"wrote {OUT}: {nmax} max, {nmin3} min3, {nmin} min, {nperm} prmt")


if __name__ == "__main__":
    main()
