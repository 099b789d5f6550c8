// hs_search_ga_spec.cu -- K3 for one GA (evolve, scheduler.py:515-574) as a
// speculative generation pipeline over a thread-block cluster.
//
// A steady-state generation is one long dependent chain (crossover, up to
// max_passes local-search passes, pricing the snapshots), but generation
// g + 1 depends on generation g only through
//   (a) the PCG64 stream position: g's parent draws, its crossover draws and
//       one permutation(C(k,2)) per sweep pass that ran (_pass_ours even
//       phases, :405-412; the chain and KL passes draw nothing), and
//   (b) the population: g replaces the first-maximum member if its best
//       snapshot is cheaper (:555-567).
// CTA 0's warp 0 (the sequencer) therefore runs ahead: it draws g + 1's
// parents and replays its crossover on the committed population, advances
// the stream by the number of sweep passes the previous generation used
// (the prediction; constant over a run on every paper scenario), and hands
// the job (parents + stream state) to an idle worker CTA through distributed
// shared memory.  Workers run the unchanged refine / pricing code (sweep
// waves over their 8 warps, register chain rounds, warp pricing) and post
// the best snapshot back.  The sequencer commits generations strictly in
// order with the reference's selection rules.  Two things can invalidate a
// job already in flight, and both are checked at commit: a wrong sweep-count
// prediction for the committing generation (every later job started from a
// wrong stream position), and a replacement of a member that a later job
// took as a parent (that job and every later one: their crossover draws
// depend on the parents).  Replacements are rare (6% of the generations of
// the 1000-generation anchors), so jobs are issued optimistically; the
// invalid ones are drained and re-issued from the recorded stream state.
// A patience stop drains everything after it.  Results, traces, evaluation
// counts and the final stream state are exactly those of the sequential
// kernel.
#include <cooperative_groups.h>

#include "hs_search_impl.cuh"

namespace cg = cooperative_groups;

namespace hs {

constexpr int kSpecMaxKM = 128;     // layouts of up to 128 devices on this path
constexpr int kSpecMaxCluster = 16;

struct SpecJob {  // in each worker's shared memory, written by the sequencer
    int seq, gen, pad0, pad1;
    hs_pcg64 rng;  // after the parent draws (the worker replays the crossover)
    int16_t par[2 * kSpecMaxKM];
};

struct SpecRes {  // in CTA 0's shared memory, one per worker, written by the worker
    int seq, nsnap, draws, pad;
    double cost;   // the best snapshot's total (first strict minimum)
    hs_pcg64 rng;  // after the refine
    int16_t lay[kSpecMaxKM];
};

size_t spec_extra_bytes() {
    return ((sizeof(SpecJob) + 15) & ~(size_t)15) + ((sizeof(SpecRes) * kSpecMaxCluster + 15) & ~(size_t)15) + 64;
}

__device__ __forceinline__ void st_release_cluster(int* p, int v) {
    asm volatile("st.release.cluster.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire_cluster(const int* p) {
    int v;
    asm volatile("ld.acquire.cluster.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }

// The stream consumption of crossover(p1, p2, rng) (scheduler.py:139-174)
// without building the child: the draws depend on the parents only through
// the number of differing slots, the chosen slot's |diff| and the drawn
// subset size.  Same calls, same order as crossover() (hs_search_impl.cuh).
__device__ __noinline__ void crossover_draws(LS& s, const int16_t* p1, const int16_t* p2, Pcg64& rng, int lane) {
    const int k = s.k, m = s.m;
    for (int t = lane; t < k * m; t += kWarp) s.grp_of[p1[t]] = (int8_t)(t / m);
    __syncwarp();
    // lane j < k: |diff_j| = members of p2's group j outside p1's group j
    int c = 0;
    if (lane < k)
        for (int i = 0; i < m; i++) c += s.grp_of[p2[lane * m + i]] != lane;
    const unsigned nz = __ballot_sync(kFull, lane < k && c > 0);
    int cnts[16];
#pragma unroll
    for (int j = 0; j < 16; j++) cnts[j] = __shfl_sync(kFull, c, j);
    if (lane == 0) {
        const int ns = __popc(nz);
        if (ns > 0) {
            const int pick = (int)rng.integers(0, ns);
            int j = 0;
            for (unsigned b = nz, q = 0;; b &= b - 1, q++) {
                if ((int)q == pick) {
                    j = __ffs(b) - 1;
                    break;
                }
            }
            int nd = 0;
#pragma unroll
            for (int x = 0; x < 16; x++) nd = x == j ? cnts[x] : nd;
            const int mi = (int)rng.integers(1, nd + 1);
            for (int jj = nd - mi; jj < nd; jj++) (void)rng.bounded((uint64_t)jj);  // Floyd
            for (int i = mi - 1; i >= 1; i--) (void)rng.bounded((uint64_t)i);       // shuffle
            for (int t = 0; t < mi; t++) (void)rng.integers(0, m - t);              // evictions
        }
    }
    __syncwarp();
}

template <bool kSmemTables, typename KeyT, bool kM8>
__global__ void __launch_bounds__(256) ga_spec_kernel(GAArgs a, ScratchLayout wl) {
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank(), C = (int)cl.num_blocks(), NW = C - 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int n = a.n, k = a.k, m = kM8 ? 8 : a.m, km = k * m, P = a.pop, cap = m + 1;
    const int max_snaps = 1 + a.max_passes;
    size_t off = 0;
    const Pricer<KeyT, kM8, false> pr = make_pricer<kSmemTables, KeyT, kM8, false>(
        n, k, m, a.dp, a.rank, a.vals, a.hk, a.hkb, a.hk_scratch, a.hk_size, wl, smem, off, wid, W);
    const double* SW;
    if (kSmemTables) {
        double* ssw = reinterpret_cast<double*>(smem + off);
        off += (size_t)n * n * 8;
        for (int i = threadIdx.x; i < n * n; i += blockDim.x) ssw[i] = a.sw[i];
        SW = ssw;
    } else {
        SW = a.sw;
    }
    auto take = [&](size_t bytes) {
        unsigned char* p = smem + off;
        off += (bytes + 15) & ~(size_t)15;
        return p;
    };
    GASmem g;
    g.snaps = reinterpret_cast<int16_t*>(take((size_t)max_snaps * km * 2));
    g.snapcost = reinterpret_cast<double*>(take((size_t)max_snaps * 8));
    g.popcost = reinterpret_cast<double*>(take((size_t)P * 8));
    g.best = reinterpret_cast<int16_t*>(take((size_t)km * 2));
    g.par = reinterpret_cast<int16_t*>(take((size_t)2 * km * 2));
    g.ctl = reinterpret_cast<int*>(take(16 * 4));
    LS& s = g.ls;
    s.n = n;
    s.k = k;
    s.m = m;
    s.cap = cap;
    s.W = SW;
    s.w_sh = kSmemTables ? (uint32_t)__cvta_generic_to_shared(SW) : 0u;
    s.lat = true;
    s.G = reinterpret_cast<int16_t*>(take((size_t)k * cap * 2));
    s.sz = reinterpret_cast<int*>(take((size_t)k * 4));
    s.mean = reinterpret_cast<double*>(take((size_t)n * k * 8));
    s.mver = reinterpret_cast<uint32_t*>(take((size_t)n * k * 4));
    s.cver = reinterpret_cast<uint32_t*>(take((size_t)k * 4));
    s.home = reinterpret_cast<double*>(take((size_t)n * 8));
    s.valid = reinterpret_cast<int*>(take(16));
    s.fe = reinterpret_cast<int16_t*>(take((size_t)k * 4));
    s.bpv = reinterpret_cast<double*>(take((size_t)n * 8));
    s.bpp = reinterpret_cast<int16_t*>(take((size_t)n * 2));
    s.locked = reinterpret_cast<uint32_t*>(take((size_t)((n + 31) >> 5) * 4));
    s.nlocked = reinterpret_cast<int*>(take(4));
    s.perm = reinterpret_cast<int16_t*>(take((size_t)(k * k + cap) * 2));
    s.f64 = reinterpret_cast<double*>(take((size_t)(4 * cap + 2 * k + 2) * 8));
    s.i32 = reinterpret_cast<int*>(take((size_t)(3 * k + 8) * 4));
    s.grp_of = reinterpret_cast<int8_t*>(take((size_t)n));
    GAState* stp = reinterpret_cast<GAState*>(take(sizeof(GAState)));
    SpecJob* job = reinterpret_cast<SpecJob*>(take(sizeof(SpecJob)));
    SpecRes* res = reinterpret_cast<SpecRes*>(take(sizeof(SpecRes) * kSpecMaxCluster));
    for (int t = threadIdx.x; t < n * k; t += blockDim.x) s.mver[t] = 0;
    for (int t = threadIdx.x; t < k; t += blockDim.x) s.cver[t] = 1;
    if (threadIdx.x == 0) job->seq = -2;
    if (threadIdx.x < kSpecMaxCluster) res[threadIdx.x].seq = -2;
    __syncthreads();
    cl.sync();  // every mailbox is initialised before anyone posts to it

    int16_t* pop = a.pop_buf;
    double* gcost = a.cost_buf;
    int16_t* gbest = a.best_buf;
    const int np = k * (k - 1) / 2;
    const bool waves = a.kind == 0 && m == 8 && n <= 128 && W > 1;
    const int stop_after = a.kind == 0 ? 2 : 1;

    if (rank == 0) {
        if (wid == 0) {
            // ------------------------------------------------------------ sequencer
            GAState& st = *stp;
            if (lane == 0) st = a.state[0];
            __syncwarp();
            for (int t = lane; t < P; t += kWarp) g.popcost[t] = gcost[t];
            __syncwarp();
            const int gen_end = min(a.gen_end, a.generations);
            Pcg64 rs;                  // speculative stream: the next job's parent draws start here
            if (lane == 0) rs.load(st.rng);
            hs_pcg64 rcommit = st.rng;  // stream after the last committed generation
            int pred = (a.kind == 0 && m >= 2) ? (a.max_passes + 1) / 2 : 0;
            int gen_c = st.gen, gen_s = st.gen, seqctr = 0;
            bool stopping = st.stopped != 0;
            int wseq[kSpecMaxCluster], wstate[kSpecMaxCluster];  // state: 0 free, 1 live job, 2 draining
            // per in-flight generation (index gen % 16): worker, predicted sweep
            // draws, parent slots, stream state before its parent draws
            int ring[kSpecMaxCluster], assumed[kSpecMaxCluster], par1[kSpecMaxCluster], par2[kSpecMaxCluster];
            hs_pcg64 start[kSpecMaxCluster];
            for (int x = 0; x < kSpecMaxCluster; x++) wseq[x] = wstate[x] = ring[x] = assumed[x] = par1[x] = par2[x] = 0;
            for (;;) {
                int act = 0, w = -1;
                if (lane == 0) {
                    for (int x = 0; x < NW; x++)
                        if (wstate[x] == 2 && ld_acquire_cluster(&res[x].seq) == wseq[x]) wstate[x] = 0;
                    if (gen_c < gen_s) {
                        const int x = ring[gen_c % kSpecMaxCluster];
                        if (ld_acquire_cluster(&res[x].seq) == wseq[x]) {
                            act = 1;
                            w = x;
                        }
                    }
                    if (!act) {
                        if (stopping || gen_c >= gen_end) {
                            bool idle = gen_c == gen_s;
                            for (int x = 0; x < NW; x++) idle = idle && wstate[x] == 0;
                            if (idle) act = 3;
                        } else if (gen_s < gen_end && gen_s - gen_c < NW) {
                            for (int x = 0; x < NW && w < 0; x++)
                                if (wstate[x] == 0) w = x;
                            if (w >= 0) act = 2;
                        }
                    }
                }
                act = __shfl_sync(kFull, act, 0);
                w = __shfl_sync(kFull, w, 0);
                if (act == 3) break;
                if (act == 0) {
                    __nanosleep(64);
                    continue;
                }
                if (act == 1) {
                    // commit generation gen_c (scheduler.py:551-567)
                    (void)ld_acquire_cluster(&res[w].seq);  // every lane reads the posted result
                    const SpecRes& R = res[w];
                    int worst = 0, replace = 0, improve = 0;
                    if (lane == 0) {
                        const int g0 = gen_c;
                        wstate[w] = 0;
                        const bool mispredicted = R.draws != assumed[g0 % kSpecMaxCluster];
                        const double cb = R.cost;
                        st.evaluations += R.nsnap;
                        for (int t = 1; t < P; t++)
                            if (g.popcost[t] > g.popcost[worst]) worst = t;  // first maximum
                        replace = cb < g.popcost[worst];
                        improve = cb < st.best_total;
                        if (replace) g.popcost[worst] = cb;
                        if (improve) {
                            st.best_total = cb;
                            st.since = 0;
                        } else {
                            st.since++;
                        }
                        if (a.trace_best) a.trace_best[g0] = st.best_total;
                        if (a.trace_mean) a.trace_mean[g0] = pw_array(g.popcost, P) / (double)P;
                        st.gen = g0 + 1;
                        gen_c = g0 + 1;
                        rcommit = R.rng;
                        if (a.patience > 0 && st.since >= a.patience) {
                            st.stopped = 1;
                            stopping = true;
                        }
                        // first later in-flight job that is no longer valid
                        int bad = gen_s;
                        if (mispredicted || stopping) {
                            bad = gen_c;  // wrong stream position for all of them / past the stop
                        } else if (replace) {
                            for (int q = gen_c; q < gen_s && bad == gen_s; q++)
                                if (par1[q % kSpecMaxCluster] == worst || par2[q % kSpecMaxCluster] == worst) bad = q;
                        }
                        if (bad < gen_s) {  // drain those jobs, re-issue from `bad`
                            for (int q = bad; q < gen_s; q++) wstate[ring[q % kSpecMaxCluster]] = 2;
                            if (bad == gen_c) {
                                rs.load(rcommit);
                            } else {
                                rs.load(start[bad % kSpecMaxCluster]);
                            }
                            gen_s = bad;
                            if (mispredicted) pred = R.draws;
                        }
                    }
                    worst = __shfl_sync(kFull, worst, 0);
                    replace = __shfl_sync(kFull, replace, 0);
                    improve = __shfl_sync(kFull, improve, 0);
                    if (replace) copy16(pop + (size_t)worst * km, R.lay, km, lane);
                    if (improve) copy16(gbest, R.lay, km, lane);
                    __syncwarp();
                    continue;
                }
                // act == 2: issue generation gen_s on worker w (parents from the
                // committed population; checked against later replacements at commit)
                int i = 0, i2 = 0;
                Pcg64 t = rs;
                hs_pcg64 after_parents;
                if (lane == 0) {
                    t.store(start[gen_s % kSpecMaxCluster]);
                    i = (int)t.integers(0, P);
                    i2 = (int)t.integers(0, P - 1);
                    if (i2 >= i) i2++;
                    t.store(after_parents);
                    par1[gen_s % kSpecMaxCluster] = i;
                    par2[gen_s % kSpecMaxCluster] = i2;
                }
                i = __shfl_sync(kFull, i, 0);
                i2 = __shfl_sync(kFull, i2, 0);
                copy16(g.par, pop + (size_t)i * km, km, lane);
                copy16(g.par + km, pop + (size_t)i2 * km, km, lane);
                __syncwarp();
                // the crossover's stream consumption (depends on the parents)
                crossover_draws(s, g.par, g.par + km, t, lane);
                SpecJob* jw = cl.map_shared_rank(job, w + 1);
                for (int q = lane; q < 2 * km; q += kWarp) jw->par[q] = g.par[q];
                if (lane == 0) {
                    for (int p = 0; p < pred; p++)
                        for (int q = np - 1; q >= 1; q--) (void)t.interval((uint64_t)q);
                    rs = t;
                    jw->gen = gen_s;
                    jw->rng = after_parents;
                    assumed[gen_s % kSpecMaxCluster] = pred;
                    ring[gen_s % kSpecMaxCluster] = w;
                    wstate[w] = 1;
                    wseq[w] = ++seqctr;
                    gen_s++;
                }
                fence_cluster();
                __syncwarp();
                if (lane == 0) st_release_cluster(&jw->seq, seqctr);
            }
            // workers are idle: release them, persist the committed state
            for (int x = lane; x < NW; x += kWarp) st_release_cluster(&cl.map_shared_rank(job, x + 1)->seq, -1);
            for (int q = lane; q < P; q += kWarp) gcost[q] = g.popcost[q];
            if (lane == 0) {
                st.rng = rcommit;
                a.state[0] = st;
            }
        }
    } else {
        // -------------------------------------------------------------- worker
        SpecRes* R = cl.map_shared_rank(res, 0) + (rank - 1);
        const bool driver = wid == 0;
        int last = -2;
        for (;;) {
            if (threadIdx.x == 0) {
                int sq;
                while ((sq = ld_acquire_cluster(&job->seq)) == last) __nanosleep(32);
                last = sq;
                g.ctl[4] = sq;
            }
            __syncthreads();
            const int sq = g.ctl[4];
            if (sq < 0) break;
            (void)ld_acquire_cluster(&job->seq);  // every thread reads the posted job
            for (int q = threadIdx.x; q < 2 * km; q += blockDim.x) g.par[q] = job->par[q];
            Pcg64 rng;
            if (driver) rng.load(job->rng);
            __syncthreads();
            int draws = 0;
            if (driver) {
                crossover(s, g.par, g.par + km, rng, g.snaps, lane);
                int nsnap = 1;
                if (a.kind != 2 && !waves) {  // _refine (:455-487) on the driver warp
                    load_groups(s, g.snaps, lane);
                    int stale = 0;
                    for (int t = 0; t < a.max_passes; t++) {
                        bool changed;
                        if (a.kind == 0) {
                            if (s.sz[0] < 2) {
                                changed = false;
                            } else if (t % 2 == 0) {
                                draws++;
                                changed = pass_sweep(s, rng, lane);
                            } else {
                                changed = pass_chains(s, lane);
                            }
                        } else {
                            changed = pass_kl(s, lane);
                        }
                        if (!changed) {
                            if (++stale >= stop_after) break;
                            continue;
                        }
                        stale = 0;
                        store_groups(s, g.snaps + (size_t)nsnap * km, lane);
                        nsnap++;
                    }
                }
                if (waves) load_groups(s, g.snaps, lane);
                if (lane == 0) g.ctl[0] = nsnap;
            }
            if (waves) {
                __syncthreads();
                int nsnap = 1, stale = 0;
                for (int t = 0; t < a.max_passes; t++) {
                    bool changed;
                    if (t % 2 == 0) {
                        draws++;
                        changed = s.w_sh ? pass_sweep_waves<true>(s, rng, wid, lane, W, g.ctl + 3)
                                         : pass_sweep_waves<false>(s, rng, wid, lane, W, g.ctl + 3);
                    } else {
                        if (driver) {
                            const bool ch = pass_chains(s, lane);
                            if (lane == 0) g.ctl[3] = ch;
                        }
                        __syncthreads();
                        changed = g.ctl[3] != 0;
                    }
                    __syncthreads();
                    if (!changed) {
                        if (++stale >= stop_after) break;
                        continue;
                    }
                    stale = 0;
                    if (driver) store_groups(s, g.snaps + (size_t)nsnap * km, lane);
                    nsnap++;
                }
                if (threadIdx.x == 0) g.ctl[0] = nsnap;
            }
            __syncthreads();
            const int nsnap = g.ctl[0];
            pr.all(g.snaps, nsnap, km, g.snapcost, wid, W, lane);
            __syncthreads();
            if (driver) {
                int bsi = 0;
                if (lane == 0)
                    for (int q = 1; q < nsnap; q++)
                        if (g.snapcost[q] < g.snapcost[bsi]) bsi = q;  // first strict minimum
                bsi = __shfl_sync(kFull, bsi, 0);
                copy16(R->lay, g.snaps + (size_t)bsi * km, km, lane);
                if (lane == 0) {
                    R->cost = g.snapcost[bsi];
                    R->nsnap = nsnap;
                    R->draws = draws;
                    rng.store(R->rng);
                }
                fence_cluster();
                __syncwarp();
                if (lane == 0) st_release_cluster(&R->seq, sq);
            }
            __syncthreads();
        }
    }
    __syncthreads();
    cl.sync();  // no CTA leaves while a peer may still touch its shared memory
}

template <bool S, typename KT, bool M8>
static int launch_spec_t(const GAArgs& a, const SearchPlan& plan, int cluster, cudaStream_t st) {
    ScratchLayout wl = scratch_layout(a.k <= 8 ? a.k : 8, a.m);
    const size_t smem = plan.smem + spec_extra_bytes();
    auto kern = ga_spec_kernel<S, KT, M8>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
    if (cluster > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster);
    cfg.blockDim = dim3(plan.warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, wl) == cudaSuccess ? 0 : -1;
}

template <bool S, typename KT, bool M8>
static int spec_cluster_t(const SearchPlan& plan) {
    const size_t smem = plan.smem + spec_extra_bytes();
    auto kern = ga_spec_kernel<S, KT, M8>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {16, 8, 4}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c);
        cfg.blockDim = dim3(plan.warps * 32);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = c;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) == cudaSuccess && nc >= 1) return c;
        cudaGetLastError();
    }
    return 0;
}

// Cluster size for the speculative GA of this plan (0: not available).
int ga_spec_cluster(const GAArgs& a, const SearchPlan& plan, bool key16, size_t smem_optin) {
    if (plan.cta || plan.warp_islands || a.n > kSpecMaxKM || a.k > 8 || plan.warps < 2) return 0;
    if (plan.smem + spec_extra_bytes() > smem_optin) return 0;
    if (plan.m8) return plan.smem_tables ? spec_cluster_t<true, uint16_t, true>(plan)
                                         : spec_cluster_t<false, uint16_t, true>(plan);
    if (key16) return plan.smem_tables ? spec_cluster_t<true, uint16_t, false>(plan)
                                       : spec_cluster_t<false, uint16_t, false>(plan);
    return plan.smem_tables ? spec_cluster_t<true, uint32_t, false>(plan) : spec_cluster_t<false, uint32_t, false>(plan);
}

int launch_ga_spec(const GAArgs& a, const SearchPlan& plan, int cluster, bool key16, cudaStream_t st) {
    if (plan.m8) return plan.smem_tables ? launch_spec_t<true, uint16_t, true>(a, plan, cluster, st)
                                         : launch_spec_t<false, uint16_t, true>(a, plan, cluster, st);
    if (key16) return plan.smem_tables ? launch_spec_t<true, uint16_t, false>(a, plan, cluster, st)
                                       : launch_spec_t<false, uint16_t, false>(a, plan, cluster, st);
    return plan.smem_tables ? launch_spec_t<true, uint32_t, false>(a, plan, cluster, st)
                            : launch_spec_t<false, uint32_t, false>(a, plan, cluster, st);
}

}  // namespace hs
