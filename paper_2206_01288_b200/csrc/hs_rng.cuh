// hs_rng.cuh -- numpy Generator(PCG64) on the device, draw for draw.
//
// The GA consumes one sequential stream whose draw count is data-dependent
// (Lemire / masked rejection, crossover and pass counts), so the stream is
// stepped exactly like numpy does (scheduler.py:118,157-170,411,549-550):
//   next64     : 128-bit LCG step, XSL-RR output of the new state
//   next32     : buffered upper half (Generator's has_uint32 / uinteger)
//   bounded    : random_bounded_uint64, Lemire on 32-bit draws  (integers, choice)
//   interval   : random_interval, masked rejection            (permutation)
#pragma once
#include <cstdint>

#include "../../include/hetsched_b200.h"

namespace hs {

struct Pcg64 {
    uint64_t sh, sl, ih, il;
    int has32;
    uint32_t u32;

    __device__ __forceinline__ void load(const hs_pcg64& s) {
        sh = s.state_hi;
        sl = s.state_lo;
        ih = s.inc_hi;
        il = s.inc_lo;
        has32 = s.has_uint32;
        u32 = s.uinteger;
    }
    __device__ __forceinline__ void store(hs_pcg64& s) const {
        s.state_hi = sh;
        s.state_lo = sl;
        s.inc_hi = ih;
        s.inc_lo = il;
        s.has_uint32 = has32;
        s.uinteger = u32;
    }
    __device__ __forceinline__ uint64_t next64() {
        const uint64_t MH = 0x2360ED051FC65DA4ull, ML = 0x4385DF649FCCF645ull;
        uint64_t lo = sl * ML;
        uint64_t hi = __umul64hi(sl, ML) + sh * ML + sl * MH;
        uint64_t nlo = lo + il;
        hi += ih + (nlo < lo ? 1ull : 0ull);
        sl = nlo;
        sh = hi;
        uint64_t x = sh ^ sl;
        unsigned rot = (unsigned)(sh >> 58);
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    __device__ __forceinline__ uint32_t next32() {
        if (has32) {
            has32 = 0;
            return u32;
        }
        uint64_t v = next64();
        has32 = 1;
        u32 = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    // uniform on [0, rng] inclusive; rng < 2^32 on every call site here
    __device__ __forceinline__ uint64_t bounded(uint64_t rng) {
        if (rng == 0) return 0;
        if (rng == 0xFFFFFFFFull) return next32();
        uint32_t ex = (uint32_t)rng + 1u;
        uint64_t prod = (uint64_t)next32() * ex;
        uint32_t left = (uint32_t)prod;
        if (left < ex) {
            uint32_t thr = (0xFFFFFFFFu - (uint32_t)rng) % ex;
            while (left < thr) {
                prod = (uint64_t)next32() * ex;
                left = (uint32_t)prod;
            }
        }
        return prod >> 32;
    }
    __device__ __forceinline__ uint64_t interval(uint64_t mx) {
        if (mx == 0) return 0;
        uint64_t mask = mx;
        mask |= mask >> 1;
        mask |= mask >> 2;
        mask |= mask >> 4;
        mask |= mask >> 8;
        mask |= mask >> 16;
        mask |= mask >> 32;
        uint64_t v;
        while ((v = (next32() & mask)) > mx) {
        }
        return v;
    }
    // Generator.integers(low, high) with int64 output
    __device__ __forceinline__ int64_t integers(int64_t low, int64_t high) {
        return low + (int64_t)bounded((uint64_t)(high - low - 1));
    }
};

}  // namespace hs
