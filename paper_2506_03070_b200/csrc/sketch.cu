// sketch.cu -- K1 sparse-sign generation and K2 sketch apply (sm_100a).
//
// K1 replaces sketch.hpp:75-94 (rejection_sample_one), sketch.hpp:149-173
// (sparse_sign_block) and sketch.hpp:178-194 (generate_sparse_sign), bit-exact.
// Layout: one warp holds 32/G sketch columns, G = next_pow2(zeta) lanes per
// column, lane i computing draw i of the column's index substream directly
// (Weyl counter, rng.cuh).  A shuffle bitonic network sorts the G draws, a
// shfl_up comparison + __ballot_sync finds duplicates; columns with a
// duplicate (or a Lemire rejection) are replayed exactly by the group leader
// (the reference's left-to-right redraw loop), which happens for ~zeta^2/d of
// the columns (0.7% at d=4000, zeta=8).
//
// K2 replaces csc_matrix.hpp:103-120 (spmm(csc, dense)) + csc_matrix.hpp:71-82
// (S b): Y_aug = S [A | b].  The sketch entries are bucketed once per chunk of
// K rows of A ("chunk-CSR": entries sorted by (target row r, k)).  Two gathers:
//   * exact mode (gather_kernel): each CTA owns a W-column slab of Y_aug held
//     in REGISTERS (thread t owns Y rows t, t+1024, ...) and streams its slab
//     of A through shared memory (TMA / cp.async double buffer); every Y
//     element is accumulated by one thread in ascending k -- the reference's
//     order -- with IEEE mul then add, so one split reproduces the reference Y
//     bit for bit;
//   * fast mode (gather_dmma_kernel, K2d): the chunk's entries are regrouped
//     per 8-row tile (tile_repack_kernel) and applied on the FP64 tensor cores
//     (see the K2d section below).
// No atomics anywhere; both are deterministic.
#include <algorithm>
#include <cmath>
#include <cstring>

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ptx.cuh"
#include "rng.cuh"
#include "sketch.cuh"

namespace cg = cooperative_groups;

namespace slq {

namespace {

constexpr uint32_t kPad = 0xFFFFFFFFu;

struct GenArgs {
    int64_t d, zeta, col_begin, ncols;
    uint64_t seed_mixed, thresh;
    double val;
    uint32_t* compact;
    int64_t* rows64;
    double* vals;
    int64_t* colptr;
    unsigned long long* stats;
};

template <class T>
__device__ void insertion_sort(T* a, int64_t n) {
    for (int64_t i = 1; i < n; ++i) {
        T v = a[i];
        int64_t j = i - 1;
        while (j >= 0 && a[j] > v) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = v;
    }
}

template <class T>
__device__ void heap_sort(T* a, int64_t n) {
    auto sift = [&](int64_t start, int64_t end) {
        int64_t root = start;
        while (2 * root + 1 <= end) {
            int64_t child = 2 * root + 1, sw = root;
            if (a[sw] < a[child]) sw = child;
            if (child + 1 <= end && a[sw] < a[child + 1]) sw = child + 1;
            if (sw == root) return;
            T t = a[root];
            a[root] = a[sw];
            a[sw] = t;
            root = sw;
        }
    };
    for (int64_t s = (n - 2) / 2; s >= 0; --s) sift(s, n - 1);
    for (int64_t e = n - 1; e > 0; --e) {
        T t = a[0];
        a[0] = a[e];
        a[e] = t;
        sift(0, e - 1);
    }
}

template <class T>
__device__ __forceinline__ void sort_small(T* a, int64_t n) {
    if (n <= 64) insertion_sort(a, n);
    else heap_sort(a, n);
}

// sketch.hpp:75-94, sequential, on an array of T.  Returns resampled flag.
template <class T>
__device__ bool replay_column(T* out, int64_t zeta, uint64_t d, uint64_t thresh, uint64_t s0,
                              unsigned long long* rounds) {
    SeqRng rng{s0};
    for (int64_t i = 0; i < zeta; ++i) out[i] = static_cast<T>(rng.below(d, thresh));
    sort_small(out, zeta);
    bool resampled = false;
    for (;;) {
        int64_t bad = 0;
        for (int64_t i = 1; i < zeta; ++i) {
            if (out[i] == out[i - 1]) {
                out[i] = static_cast<T>(rng.below(d, thresh));
                ++bad;
            }
        }
        if (bad == 0) break;
        resampled = true;
        ++(*rounds);
        sort_small(out, zeta);
    }
    return resampled;
}

// Warp-group generator: G lanes per column (zeta <= G <= 32), d < 2^31.
template <int G>
__global__ void __launch_bounds__(256) gen_warp_kernel(GenArgs a) {
    constexpr int kCols = 32 / G;
    __shared__ uint32_t fb[8][32];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int gl = lane & (G - 1);
    const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t j = gwarp * kCols + lane / G;
    const bool col_ok = j < a.ncols;
    const bool active = col_ok && gl < a.zeta;
    const uint64_t gj = static_cast<uint64_t>(a.col_begin + (col_ok ? j : 0));

    const uint64_t s_idx = stream_state(a.seed_mixed, 2 * gj);
    bool rej = false;
    uint32_t key = kPad;
    if (active) key = static_cast<uint32_t>(lemire(draw_at(s_idx, gl + 1), a.d, a.thresh, rej));
    rej = rej && active;

    // bitonic sort of G keys within the group (ascending, pads last)
#pragma unroll
    for (int k = 2; k <= G; k <<= 1) {
#pragma unroll
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            uint32_t other = __shfl_xor_sync(0xffffffffu, key, jj);
            const bool up = (gl & k) == 0;
            const bool lower = (gl & jj) == 0;
            key = (lower == up) ? min(key, other) : max(key, other);
        }
    }
    uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1, G);
    const bool dup = active && gl > 0 && key == prev;
    const unsigned bal = __ballot_sync(0xffffffffu, dup || rej);
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const bool need = (bal & gmask) != 0;
    if (__any_sync(0xffffffffu, need)) {
        if (need && gl == 0) {
            uint32_t* buf = &fb[wib][lane];
            unsigned long long rounds = 0;
            bool res = replay_column(buf, a.zeta, a.d, a.thresh, s_idx, &rounds);
            if (a.stats) {
                if (res) atomicAdd(&a.stats[0], 1ull);
                if (rounds) atomicAdd(&a.stats[1], rounds);
            }
        }
        __syncwarp();
        if (need && active) key = fb[wib][(lane & ~(G - 1)) + gl];
        __syncwarp();
    }
    if (!active) return;
    // sketch.hpp:168-169: sign i (drawn in order from stream 2j+1) pairs with
    // the i-th smallest row.
    const uint64_t s_val = stream_state(a.seed_mixed, 2 * gj + 1);
    const bool pos = draw_at(s_val, gl + 1) & 1u;
    const int64_t e = j * a.zeta + gl;
    if (a.compact) a.compact[e] = key | (pos ? 0u : 0x80000000u);
    if (a.rows64) a.rows64[e] = key;
    if (a.vals) a.vals[e] = pos ? a.val : -a.val;
    if (a.colptr) {
        if (gl == 0) a.colptr[j + 1] = (j + 1) * a.zeta;
        if (j == 0 && gl == 0) a.colptr[0] = 0;
    }
}

// Generic path (zeta > 32 or huge d): one thread per column, sequential
// replay on an int64 work array (rows64, always provided by the host).
__global__ void gen_generic_kernel(GenArgs a) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= a.ncols) return;
    const uint64_t gj = static_cast<uint64_t>(a.col_begin + j);
    int64_t* rows = a.rows64 + j * a.zeta;
    unsigned long long rounds = 0;
    bool res = replay_column(rows, a.zeta, a.d, a.thresh, stream_state(a.seed_mixed, 2 * gj), &rounds);
    if (a.stats) {
        if (res) atomicAdd(&a.stats[0], 1ull);
        if (rounds) atomicAdd(&a.stats[1], rounds);
    }
    SeqRng vr{stream_state(a.seed_mixed, 2 * gj + 1)};
    for (int64_t i = 0; i < a.zeta; ++i) {
        const bool pos = vr.next() & 1u;
        if (a.vals) a.vals[j * a.zeta + i] = pos ? a.val : -a.val;
        if (a.compact) a.compact[j * a.zeta + i] = static_cast<uint32_t>(rows[i]) | (pos ? 0u : 0x80000000u);
    }
    if (a.colptr) {
        a.colptr[j + 1] = (j + 1) * a.zeta;
        if (j == 0) a.colptr[0] = 0;
    }
}

// Synthetic sparse rows for the C4 benchmark harness: row i
// (global id g) gets nnz distinct columns of [0, n) drawn by the reference's
// rejection sampler from substream (seed, 2g) -- sorted -- and values
// +-scale[col] with signs from substream (seed, 2g+1).
__global__ void sparse_rows_kernel(int64_t n, int64_t nnz, uint64_t seed_mixed, uint64_t thresh, int64_t row_begin,
                                   int64_t m, const double* scale, int64_t* rowptr, int32_t* colidx, double* vals,
                                   int64_t* work) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > m) return;
    rowptr[i] = i * nnz;
    if (i == m) return;
    const uint64_t g = static_cast<uint64_t>(row_begin + i);
    int64_t* cols = work + i * nnz;
    unsigned long long rounds = 0;
    replay_column(cols, nnz, static_cast<uint64_t>(n), thresh, stream_state(seed_mixed, 2 * g), &rounds);
    SeqRng vr{stream_state(seed_mixed, 2 * g + 1)};
    for (int64_t t = 0; t < nnz; ++t) {
        const int64_t c = cols[t];
        colidx[i * nnz + t] = static_cast<int32_t>(c);
        const double sg = (vr.next() & 1u) ? 1.0 : -1.0;
        vals[i * nnz + t] = scale ? sg * scale[c] : sg;
    }
}

// ------------------------------------------------------------- K2 bucketize

struct BucketArgs {
    const uint32_t* compact;
    const int64_t* colptr;  // null => uniform zeta
    int64_t zeta, ncols, d;
    int K, KB;
    int64_t ptr_stride, ent_stride;  // u16 units per chunk
    uint16_t* ptr_out;
    uint16_t* ent_out;
    int cap;                         // smem key capacity (power of 2)
    int* overflow;
    int slots;                       // 0: (k_local << 1 | neg); W = 4 / 2 / 1: gather_kernel byte offsets (see below)
};

__device__ __forceinline__ int gslot(int k, int h);

__global__ void __launch_bounds__(1024) bucketize_kernel(BucketArgs a) {
    extern __shared__ uint32_t keys[];
    const int tid = threadIdx.x, T = blockDim.x;
    const int64_t c = blockIdx.x;
    const int64_t k0 = c * a.K;
    const int64_t kc = min(static_cast<int64_t>(a.K), a.ncols - k0);
    const int64_t eb = a.colptr ? a.colptr[k0] : k0 * a.zeta;
    const int64_t ee = a.colptr ? a.colptr[k0 + kc] : (k0 + kc) * a.zeta;
    const int N = static_cast<int>(ee - eb);
    if (N > a.cap) {
        if (tid == 0) atomicExch(a.overflow, 1);
        return;
    }
    int NP = 2;
    while (NP < N) NP <<= 1;
    const int sh = a.KB + 1;
    if (a.colptr) {
        for (int64_t kl = tid; kl < kc; kl += T)
            for (int64_t e = a.colptr[k0 + kl]; e < a.colptr[k0 + kl + 1]; ++e) {
                const uint32_t ent = a.compact[e];
                keys[e - eb] = ((ent & 0x7fffffffu) << sh) | (static_cast<uint32_t>(kl) << 1) | (ent >> 31);
            }
    } else {
        for (int i = tid; i < N; i += T) {
            const uint32_t ent = a.compact[eb + i];
            const uint32_t kl = static_cast<uint32_t>(i / a.zeta);
            keys[i] = ((ent & 0x7fffffffu) << sh) | (kl << 1) | (ent >> 31);
        }
    }
    for (int i = N + tid; i < NP; i += T) keys[i] = kPad;
    __syncthreads();
    for (int k = 2; k <= NP; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = tid; i < (NP >> 1); i += T) {
                const int lo = ((i & ~(jj - 1)) << 1) | (i & (jj - 1));
                const int hi = lo + jj;
                const bool asc = (lo & k) == 0;
                const uint32_t x = keys[lo], y = keys[hi];
                if ((x > y) == asc) {
                    keys[lo] = y;
                    keys[hi] = x;
                }
            }
            __syncthreads();
        }
    }
    uint16_t* ent = a.ent_out + c * a.ent_stride;
    uint16_t* ptr = a.ptr_out + c * a.ptr_stride;
    const uint32_t lowmask = (1u << sh) - 1u;
    for (int i = tid; i < N; i += T) {
        const uint32_t kv = keys[i] & lowmask;  // k_local << 1 | neg
        // slots: byte offset of the entry's A row in the gather's smem stage
        // (W = 4: the first 16-byte half, the second at offset ^ 16) with the
        // sign in bit 0, so the gather decodes an entry with a few logic ops
        const int kl = static_cast<int>(kv >> 1);
        const uint32_t off = a.slots == 4 ? static_cast<uint32_t>(kl) << 5
                             : a.slots == 2 ? static_cast<uint32_t>(kl) << 4
                                            : static_cast<uint32_t>(kl) << 3;
        ent[i] = a.slots ? static_cast<uint16_t>(off | (kv & 1u)) : static_cast<uint16_t>(kv);
        const int64_t r = keys[i] >> sh;
        const int64_t rp = (i == 0) ? -1 : static_cast<int64_t>(keys[i - 1] >> sh);
        for (int64_t rr = rp + 1; rr <= r; ++rr) ptr[rr] = static_cast<uint16_t>(i);
    }
    const int64_t rl = (N == 0) ? -1 : static_cast<int64_t>(keys[N - 1] >> sh);
    for (int64_t rr = rl + 1 + tid; rr <= a.d; rr += T) ptr[rr] = static_cast<uint16_t>(N);
}

// The same chunk-CSR for a uniform zeta and slots == 0 (the sparse path's S^T
// build), by a stable counting sort instead of the bitonic network: ONE warp
// per chunk (16 KB of u16 bin counters for d <= 8192, so many chunks per SM),
// (1) bin counts with __match_any_sync (one leader per distinct row writes,
// no atomics), (2) an exclusive scan of the d counts -> the chunk's row
// pointers, (3) a second in-order walk placing each entry at its bin cursor +
// its rank among equal rows of the round: ascending k within a row, the
// bitonic sort's order exactly (its keys are (row, k) and unique).
constexpr int kBcMaxD = 8192;

__global__ void __launch_bounds__(32) bucketize_count_kernel(BucketArgs a) {
    extern __shared__ uint16_t bcnt[];  // [d]
    constexpr int kU = 8;               // rounds of entries loaded ahead (one latency per 8 rounds)
    const int lane = threadIdx.x;
    const int64_t c = blockIdx.x;
    const int64_t k0 = c * a.K;
    const int64_t kc = min(static_cast<int64_t>(a.K), a.ncols - k0);
    const int64_t eb = k0 * a.zeta;
    const int N = static_cast<int>(kc * a.zeta);
    const int d = static_cast<int>(a.d);
    if (N > a.cap) {
        if (lane == 0) atomicExch(a.overflow, 1);
        return;
    }
    for (int r = lane; r < d; r += 32) bcnt[r] = 0;
    __syncwarp();
    const uint32_t* src = a.compact + eb;
    const unsigned below = (1u << lane) - 1u;
    for (int b = 0; b < N; b += 32 * kU) {
        uint32_t e8[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) e8[u] = src[min(b + 32 * u + lane, N - 1)];  // unconditional (see sl_issue)
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const bool live = b + 32 * u + lane < N;
            const uint32_t r = live ? (e8[u] & 0x7fffffffu) : 0xffffffffu;
            const unsigned peers = __match_any_sync(0xffffffffu, r);
            if (live && (peers & below) == 0) bcnt[r] += static_cast<uint16_t>(__popc(peers));
            __syncwarp();
        }
    }
    // exclusive scan of the counts: lane l owns bins [l q, (l + 1) q)
    const int q = (d + 31) / 32;
    const int r0 = min(d, lane * q), r1 = min(d, r0 + q);
    int sum = 0;
    for (int r = r0; r < r1; ++r) sum += bcnt[r];
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    int run = x - sum;
    for (int r = r0; r < r1; ++r) {
        const int v = bcnt[r];
        bcnt[r] = static_cast<uint16_t>(run);
        run += v;
    }
    __syncwarp();
    uint16_t* ptr = a.ptr_out + c * a.ptr_stride;
    for (int r = lane; r < d; r += 32) ptr[r] = bcnt[r];  // coalesced
    if (lane == 31) ptr[d] = static_cast<uint16_t>(x);
    uint16_t* ent = a.ent_out + c * a.ent_stride;
    const int zeta = static_cast<int>(a.zeta);
    for (int b = 0; b < N; b += 32 * kU) {
        uint32_t e8[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) e8[u] = src[min(b + 32 * u + lane, N - 1)];  // unconditional (see sl_issue)
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = b + 32 * u + lane;
            const bool live = i < N;
            const uint32_t r = live ? (e8[u] & 0x7fffffffu) : 0xffffffffu;
            const unsigned peers = __match_any_sync(0xffffffffu, r);
            if (live) {
                const int pos = bcnt[r] + __popc(peers & below);
                ent[pos] = static_cast<uint16_t>((static_cast<unsigned>(i / zeta) << 1) | (e8[u] >> 31));
            }
            __syncwarp();
            if (live && (peers & below) == 0) bcnt[r] += static_cast<uint16_t>(__popc(peers));
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------- K2 gather

constexpr int kGThreads = 1024;

struct GatherArgs {
    const double* A;  // row-major block, row 0 = local row 0
    int64_t ld, m, d;
    int K;
    int64_t nchunks, nsplit;
    int64_t ptr_stride, ent_stride;
    const uint16_t* ptr;
    const uint16_t* ent;
    double val;
    int64_t ldw;   // columns of Yw (>= ld, multiple of the slab width)
    double* Yw;    // [nsplit][ldw][d]
    int64_t c_lo, c_hi;  // chunk range of this launch (split evenly over nsplit)
    int accumulate;      // 1: y starts from Yw (nsplit == 1; incremental row ranges)
};

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 16-byte half h of A-slab row k (4 columns = 32 bytes) lives at slot
// 2k + (h ^ ((k >> 2) & 1)): the first halves of random rows then spread over
// all eight 16-byte bank groups (row parity x bit 2 of k), as do the second.
__device__ __forceinline__ int gslot(int k, int h) { return 2 * k + (h ^ ((k >> 2) & 1)); }  // gslot(k,1) == gslot(k,0)^1

template <int W>
__device__ __forceinline__ void stage_chunk(const GatherArgs& g, int64_t col0, int64_t c, double* As, uint16_t* Ps,
                                            uint16_t* Es) {
    const int tid = threadIdx.x;
    const int64_t k0 = c * g.K;
    const int kc = static_cast<int>(min(static_cast<int64_t>(g.K), g.m - k0));
    const double* base = g.A + k0 * g.ld + col0;
    if (W == 4) {
        for (int p = tid; p < 2 * kc; p += kGThreads) {
            const int k = p >> 1, h = p & 1;
            cp_async16(As + 2 * gslot(k, h), base + static_cast<int64_t>(k) * g.ld + 2 * h);
        }
    } else if (W == 2) {
        for (int k = tid; k < kc; k += kGThreads) cp_async16(As + 2 * k, base + static_cast<int64_t>(k) * g.ld);
    } else {
        for (int k = tid; k < kc; k += kGThreads) cp_async8(As + k, base + static_cast<int64_t>(k) * g.ld);
    }
    const uint16_t* gp = g.ptr + c * g.ptr_stride;
    for (int p = tid; p < g.ptr_stride / 8; p += kGThreads) cp_async16(Ps + 8 * p, gp + 8 * p);
    const uint16_t* ge = g.ent + c * g.ent_stride;
    const int nent = static_cast<int>(g.ent_stride / 8);
    for (int p = tid; p < nent; p += kGThreads) cp_async16(Es + 8 * p, ge + 8 * p);
}

template <bool EXACT>
__device__ __forceinline__ double acc_step(double y, double v, double a) {
    // EXACT: the reference's y += v * a with two roundings (csc_matrix.hpp:116)
    return EXACT ? __dadd_rn(y, __dmul_rn(v, a)) : fma(v, a, y);
}

// CTA = one 4-column slab of Y_aug, all d rows in REGISTERS: thread t owns
// rows t, t+512, ... (RPT of them).  Per chunk of K rows of A the slab
// segment (K x 32 bytes), the chunk's row pointers and its entries sorted by
// (r, k) are staged by cp.async (double buffer); each thread walks its rows'
// entries in ascending k -- the reference's order -- gathering 32 bytes of A
// per entry.
template <int RPT, int W, bool EXACT>
__global__ void __launch_bounds__(kGThreads, 1) gather_kernel(const __grid_constant__ CUtensorMap tmap, GatherArgs g) {
    // W >= 2: the A slab of a chunk arrives by TMA (2D tensor map over the
    // row-major A, boxes of 256 rows x W columns) and the chunk's row pointers
    // and entries by 1D bulk copies, all issued by one thread and completing on
    // the stage's mbarrier; W == 1 (8-byte rows, below the TMA box minimum)
    // stages with cp.async.
    constexpr bool kTma = W >= 2;
    extern __shared__ __align__(128) unsigned char gsmem[];
    __shared__ __align__(8) uint64_t full[2];
    const int tid = threadIdx.x;
    const int64_t col0 = static_cast<int64_t>(blockIdx.x) * W;
    const int64_t split = blockIdx.y;
    const int64_t cb = g.c_lo + split * (g.c_hi - g.c_lo) / g.nsplit;
    const int64_t ce = g.c_lo + (split + 1) * (g.c_hi - g.c_lo) / g.nsplit;

    const size_t a_bytes = static_cast<size_t>(g.K) * W * sizeof(double);
    const size_t p_bytes = g.ptr_stride * sizeof(uint16_t);
    const size_t e_bytes = g.ent_stride * sizeof(uint16_t);
    const size_t st_bytes = (a_bytes + p_bytes + e_bytes + 127) & ~size_t(127);
    auto As = [&](int s) { return reinterpret_cast<double*>(gsmem + s * st_bytes); };
    auto Ps = [&](int s) { return reinterpret_cast<uint16_t*>(gsmem + s * st_bytes + a_bytes); };
    auto Es = [&](int s) { return reinterpret_cast<uint16_t*>(gsmem + s * st_bytes + a_bytes + p_bytes); };

    if (kTma && tid == 0) {
        ptx::mbar_init(&full[0], 1);
        ptx::mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t c, int s) {  // thread 0: TMA the chunk into stage s
        const int64_t k0 = c * g.K;
        const int kc = static_cast<int>(min(static_cast<int64_t>(g.K), g.m - k0));
        const int nbox = (kc + 255) >> 8;
        ptx::mbar_expect_tx(&full[s], static_cast<unsigned>(nbox * 256 * W * 8 + p_bytes + e_bytes));
        for (int bx = 0; bx < nbox; ++bx) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                    ptx::smem_u32(As(s) + static_cast<size_t>(bx) * 256 * W)),
                "l"(&tmap), "r"(static_cast<int>(col0)), "r"(static_cast<int>(k0 + 256 * bx)), "r"(ptx::smem_u32(&full[s]))
                : "memory");
        }
        ptx::bulk_g2s(Ps(s), g.ptr + c * g.ptr_stride, static_cast<unsigned>(p_bytes), &full[s]);
        ptx::bulk_g2s(Es(s), g.ent + c * g.ent_stride, static_cast<unsigned>(e_bytes), &full[s]);
    };

    const uint64_t vbits = static_cast<uint64_t>(__double_as_longlong(g.val));
    double y[RPT][W];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * kGThreads;
#pragma unroll
        for (int w = 0; w < W; ++w) y[q][w] = (g.accumulate && r < g.d) ? g.Yw[(col0 + w) * g.d + r] : 0.0;
    }

    if (cb < ce) {
        if (kTma) {
            if (tid == 0) issue(cb, 0);
        } else {
            stage_chunk<W>(g, col0, cb, As(0), Ps(0), Es(0));
        }
    }
    if (!kTma) cp_commit();
    for (int64_t c = cb; c < ce; ++c) {
        const int s = static_cast<int>((c - cb) & 1);
        if (kTma) {
            if (tid == 0 && c + 1 < ce) issue(c + 1, s ^ 1);  // stage s^1 was released by the last barrier
            ptx::mbar_wait(&full[s], static_cast<unsigned>(((c - cb) >> 1) & 1));
        } else {
            if (c + 1 < ce) stage_chunk<W>(g, col0, c + 1, As(s ^ 1), Ps(s ^ 1), Es(s ^ 1));
            cp_commit();
            cp_wait<1>();
            __syncthreads();
        }
        const unsigned char* A_b = reinterpret_cast<const unsigned char*>(As(s));
        const uint16_t* P_s = Ps(s);
        const uint16_t* E_s = Es(s);
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * kGThreads;
            if (r < g.d) {
                const int e0 = P_s[r], e1 = P_s[r + 1];
                for (int e = e0; e < e1; ++e) {
                    const unsigned en = E_s[e];
                    const unsigned o0 = en & 0xFFF8u;
                    const double v = __longlong_as_double(static_cast<long long>(vbits ^ (static_cast<uint64_t>(en) << 63)));
                    if (W == 4) {
                        const double2 lo = *reinterpret_cast<const double2*>(A_b + o0);
                        const double2 hi = *reinterpret_cast<const double2*>(A_b + (o0 ^ 16u));
                        y[q][0] = acc_step<EXACT>(y[q][0], v, lo.x);
                        y[q][1 % W] = acc_step<EXACT>(y[q][1 % W], v, lo.y);
                        y[q][2 % W] = acc_step<EXACT>(y[q][2 % W], v, hi.x);
                        y[q][3 % W] = acc_step<EXACT>(y[q][3 % W], v, hi.y);
                    } else if (W == 2) {
                        const double2 lo = *reinterpret_cast<const double2*>(A_b + o0);
                        y[q][0] = acc_step<EXACT>(y[q][0], v, lo.x);
                        y[q][1 % W] = acc_step<EXACT>(y[q][1 % W], v, lo.y);
                    } else {
                        y[q][0] = acc_step<EXACT>(y[q][0], v, *reinterpret_cast<const double*>(A_b + o0));
                    }
                }
            }
        }
        __syncthreads();
    }
    if (!kTma) cp_wait<0>();
    double* Y = g.Yw + split * g.ldw * g.d;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * kGThreads;
        if (r < g.d)
#pragma unroll
            for (int w = 0; w < W; ++w) Y[(col0 + w) * g.d + r] = y[q][w];
    }
}

// Y[:, j] = sum over splits, fixed order (deterministic).
__global__ void reduce_splits_kernel(const double* Yw, int64_t nsplit, int64_t d, int64_t ld,
                                     int64_t ncols, double* Y) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= d * ncols) return;
    double s = Yw[i];
    for (int64_t p = 1; p < nsplit; ++p) s = __dadd_rn(s, Yw[p * ld * d + i]);
    Y[i] = s;
}

// ------------------------------------------------- K2d tile gather (DMMA)
//
// Fast-mode S.[A b] on the FP64 tensor cores.  A CTA owns a 16-column slab of
// Y_aug for a block of 1024 rows, held as 128 8x8 row tiles x 2 column tiles
// of mma.m8n8k4 accumulators (warp w owns row tiles w, w+32, w+64, w+96).  Per
// chunk of K <= 768 rows of A, the slab segment (K x 128 B) arrives by TMA with
// the 128-byte swizzle, together with the chunk's entries for this row block
// grouped by row tile and padded to multiples of 4 (tile_repack_kernel).  One
// group of 4 entries is one k-step: A-fragment = the 8x4 block of S (entry j's
// sign * val in the row of its target, 0 elsewhere), B-fragment = the 4 A rows'
// even / odd columns gathered from shared memory with one 16-byte load, two
// DMMAs (column tiles 0 and 1).
// Every warp runs the same instruction stream (no per-lane row ownership, so
// none of the register gather's divergence), the swizzle spreads the four
// gathered rows over the banks, and the 8x zero padding of S runs on tensor
// cores that would otherwise idle.  Order of accumulation differs from the
// reference's serial order: fast mode only (exact mode keeps gather_kernel).
constexpr int kTdRows = 1024;          // Y rows per CTA (row block)
constexpr int kTdTiles = kTdRows / 8;  // 8-row tiles per row block
constexpr int kTdHdr = 136;            // u16 header: tile offsets [129], 16-byte multiple
constexpr int kTdMaxStages = 3;

struct RepackArgs {
    const uint16_t* ptr;  // chunk-CSR row pointers (u16, per chunk ptr_stride)
    const uint16_t* ent;  // chunk-CSR entries (k_local << 1 | neg)
    int64_t ptr_stride, ent_stride, d;
    int nrb, cap;
    int64_t blk_stride;   // u16 per (chunk, row block): kTdHdr + cap
    uint16_t* out;
    int* flag;
};

// one CTA per chunk: thread (rb % 8, tile) counts its tile's entries, pads to
// a multiple of 4, a per-row-block scan places it; entries are re-encoded as
// k_local | row_in_tile << 10 | valid << 13 | neg << 15 (0 = padding).
__global__ void __launch_bounds__(1024) tile_repack_kernel(RepackArgs a) {
    __shared__ int wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t c = blockIdx.x;
    const uint16_t* ptr = a.ptr + c * a.ptr_stride;
    const uint16_t* ent = a.ent + c * a.ent_stride;
    for (int rb0 = 0; rb0 < a.nrb; rb0 += 8) {
        const int rb = rb0 + tid / kTdTiles, tb = tid % kTdTiles;
        const int64_t r0 = (static_cast<int64_t>(rb) * kTdTiles + tb) * 8;
        int e0 = 0, cnt = 0;
        if (rb < a.nrb && r0 < a.d) {
            e0 = ptr[r0];
            cnt = ptr[r0 + 8 < a.d ? r0 + 8 : a.d] - e0;
        }
        const int pad = (cnt + 3) & ~3;
        int x = pad;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        const int w0 = warp & ~3;  // 4 warps per row block
        int base = 0;
        for (int q = w0; q < warp; ++q) base += wsum[q];
        const int total = wsum[w0] + wsum[w0 + 1] + wsum[w0 + 2] + wsum[w0 + 3];
        __syncthreads();
        if (rb < a.nrb) {
            const int off = base + x - pad;
            uint16_t* blk = a.out + (c * a.nrb + rb) * a.blk_stride;
            blk[tb] = static_cast<uint16_t>(off < a.cap ? off : a.cap);
            if (tb == kTdTiles - 1) blk[kTdTiles] = static_cast<uint16_t>(total < a.cap ? total : a.cap);
            if (total > a.cap) {
                if (tb == 0) atomicExch(a.flag, 1);
            } else {
                uint16_t* eo = blk + kTdHdr + off;
                int j = 0;
                for (int rr = 0; rr < 8; ++rr) {
                    const int64_t r = r0 + rr;
                    if (r >= a.d) break;
                    for (int e = ptr[r]; e < ptr[r + 1]; ++e, ++j) {
                        const unsigned kv = ent[e];
                        eo[j] = static_cast<uint16_t>((kv >> 1) | (rr << 10) | 0x2000u | ((kv & 1u) << 15));
                    }
                }
                for (; j < pad; ++j) eo[j] = 0;
            }
        }
    }
}

// Fused bucketing for K2d (uniform zeta, the device-generated sketch): one CTA
// per chunk places the chunk's K*zeta entries straight into the tile layout,
// in entry order (stable, deterministic), without the chunk-CSR round trip:
// per-warp tile histograms (u16 pairs in smem), padded tile offsets by a scan
// per row block, then each warp re-walks its entry range and places entries
// at (its base for the tile) + (rank among equal tiles in the round, by
// __match_any_sync).  d <= 16 * 1024 (2048 tiles) keeps the histograms in smem.
struct TileBucketArgs {
    const uint32_t* compact;
    int64_t zeta, ncols, d;
    int K, nrb, cap;
    int64_t blk_stride;
    uint16_t* out;
    int* flag;
};
constexpr int kTbMaxTiles = 2048;

__global__ void __launch_bounds__(1024) tile_bucketize_kernel(TileBucketArgs a) {
    extern __shared__ int tbsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntile = static_cast<int>((a.d + 7) >> 3);
    const int nhp = (ntile + 1) >> 1;                 // packed u16 pairs per warp
    int* hist = tbsm;                                 // [32][nhp] packed counts, later bases
    int* off = hist + 32 * nhp;                       // [ntile] padded offset in the row block
    int* tot = off + ntile;                           // [ntile]
    int* rbt = tot + ntile;                           // [nrb] padded total per row block
    const int64_t c = blockIdx.x;
    const int64_t k0 = c * a.K;
    const int64_t kc = min(static_cast<int64_t>(a.K), a.ncols - k0);
    const int N = static_cast<int>(kc * a.zeta);
    const uint32_t* src = a.compact + k0 * a.zeta;
    const int per = (N + 31) / 32;
    const int wb = warp * per, we = min(N, wb + per);
    for (int i = tid; i < 32 * nhp; i += 1024) hist[i] = 0;
    __syncthreads();
    int* hw = hist + warp * nhp;
    for (int e = wb + lane; e < we; e += 32) {
        const int t = static_cast<int>((src[e] & 0x7fffffffu) >> 3);
        atomicAdd(&hw[t >> 1], 1 << (16 * (t & 1)));
    }
    __syncthreads();
    auto cnt = [&](int w, int t) { return (hist[w * nhp + (t >> 1)] >> (16 * (t & 1))) & 0xffff; };
    for (int t = tid; t < ntile; t += 1024) {
        int s = 0;
        for (int w = 0; w < 32; ++w) s += cnt(w, t);
        tot[t] = s;
    }
    __syncthreads();
    // padded offsets: warp r scans row block r's 128 tiles (4 per lane)
    for (int rb = warp; rb < a.nrb; rb += 32) {
        const int t0 = rb * kTdTiles;
        int v[4], sum = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = t0 + 4 * lane + q;
            v[q] = t < ntile ? (tot[t] + 3) & ~3 : 0;
            sum += v[q];
        }
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        int run = x - sum;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = t0 + 4 * lane + q;
            if (t < ntile) off[t] = run;
            run += v[q];
        }
        if (lane == 31) rbt[rb] = x;
    }
    __syncthreads();
    // per-warp bases (in place, packed u16): base(w, t) = off[t] + counts of
    // warps < w; one thread per word (tile pair)
    for (int hp = tid; hp < nhp; hp += 1024) {
        const int ta = 2 * hp, tb2 = ta + 1;
        int runa = off[ta], runb = tb2 < ntile ? off[tb2] : 0;
        for (int w = 0; w < 32; ++w) {
            const int word = hist[w * nhp + hp];
            const int ca = word & 0xffff, cb = (word >> 16) & 0xffff;
            hist[w * nhp + hp] = (runa & 0xffff) | ((runb & 0xffff) << 16);
            runa += ca;
            runb += cb;
        }
    }
    __syncthreads();
    bool over = false;
    for (int rb = 0; rb < a.nrb; ++rb) over |= rbt[rb] > a.cap;
    if (over) {  // flag it (the caller falls back) and leave empty tiles behind
        if (tid == 0) atomicExch(a.flag, 1);
        for (int i = tid; i < a.nrb * (kTdTiles + 1); i += 1024)
            a.out[(c * a.nrb + i / (kTdTiles + 1)) * a.blk_stride + i % (kTdTiles + 1)] = 0;
        return;
    }
    // placement, entry order (warp range, then round, then lane)
    const int zeta = static_cast<int>(a.zeta);
    for (int e0 = wb; e0 < we; e0 += 32) {
        const int e = e0 + lane;
        const bool live = e < we;
        const uint32_t en = live ? src[e] : 0u;
        const int r = static_cast<int>(en & 0x7fffffffu);
        const int t = live ? (r >> 3) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, t);
        if (live) {
            const int rank = __popc(peers & ((1u << lane) - 1u));
            const int sh = 16 * (t & 1);
            const int base = (hw[t >> 1] >> sh) & 0xffff;
            const int rb = t / kTdTiles;
            const unsigned kl = static_cast<unsigned>(e / zeta);
            a.out[(c * a.nrb + rb) * a.blk_stride + kTdHdr + base + rank] =
                static_cast<uint16_t>(kl | (static_cast<unsigned>(r & 7) << 10) | 0x2000u | ((en >> 31) << 15));
            if (rank == 0) atomicAdd(&hw[t >> 1], __popc(peers) << sh);  // the group's leader advances the base
        }
        __syncwarp();
    }
    // padding and headers
    for (int t = tid; t < ntile; t += 1024) {
        uint16_t* blk = a.out + (c * a.nrb + t / kTdTiles) * a.blk_stride;
        blk[t % kTdTiles] = static_cast<uint16_t>(off[t]);
        const int pe = (tot[t] + 3) & ~3;
        for (int j = tot[t]; j < pe; ++j) blk[kTdHdr + off[t] + j] = 0;
    }
    for (int i = tid; i < a.nrb * kTdTiles; i += 1024) {  // tiles past d (last row block)
        const int t = i;
        if (t >= ntile) a.out[(c * a.nrb + t / kTdTiles) * a.blk_stride + t % kTdTiles] = static_cast<uint16_t>(rbt[t / kTdTiles]);
    }
    for (int rb = tid; rb < a.nrb; rb += 1024) a.out[(c * a.nrb + rb) * a.blk_stride + kTdTiles] = static_cast<uint16_t>(rbt[rb]);
}

struct TdArgs {
    int64_t m, d, ldw;
    int K, box;  // rows per chunk, rows per TMA box (K is a multiple of box)
    int64_t nsplit, c_lo, c_hi;
    const uint16_t* tiles;
    int64_t blk_stride;
    int nrb, ns;
    double val;
    double* Yw;  // [nsplit][ldw][d]
};

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(1024, 1) gather_dmma_kernel(const __grid_constant__ CUtensorMap tmap, TdArgs g) {
    extern __shared__ __align__(16) unsigned char tdsm[];
    __shared__ __align__(8) uint64_t full[kTdMaxStages];
    __shared__ int done[kTdMaxStages];  // warps finished with the stage's current chunk
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lr = lane & 3, lg = lane >> 2;
    // row block fastest in the grid: the CTAs reading the same A slab chunks
    // are resident together, so A streams from DRAM once (L2 serves the rest)
    const int rb = blockIdx.x;
    const int64_t col0 = static_cast<int64_t>(blockIdx.y) * 16;
    const int64_t split = blockIdx.z;
    const int64_t cb = g.c_lo + split * (g.c_hi - g.c_lo) / g.nsplit;
    const int64_t ce = g.c_lo + (split + 1) * (g.c_hi - g.c_lo) / g.nsplit;
    // stage s: [A box K x 128 B, 1024-aligned for the 128-byte swizzle][tile block]
    // align inside the shared window (keeps the compiler on ld.shared)
    unsigned char* base = tdsm + ((1024u - (ptx::smem_u32(tdsm) & 1023u)) & 1023u);
    const size_t a_bytes = static_cast<size_t>(g.K) * 128;
    const size_t t_bytes = (static_cast<size_t>(g.blk_stride) * 2 + 1023) & ~size_t(1023);
    const size_t st_bytes = a_bytes + t_bytes;
    auto As = [&](int s) { return base + s * st_bytes; };
    auto Ts = [&](int s) { return reinterpret_cast<const uint16_t*>(base + s * st_bytes + a_bytes); };
    if (tid == 0) {
        for (int s = 0; s < g.ns; ++s) {
            ptx::mbar_init(&full[s], 1);
            done[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t c, int s) {  // one thread
        const int64_t k0 = c * g.K;
        const int kc = static_cast<int>(min(static_cast<int64_t>(g.K), g.m - k0));
        const int nbox = (kc + g.box - 1) / g.box;
        const unsigned tb = static_cast<unsigned>(g.blk_stride * 2);
        ptx::mbar_expect_tx(&full[s], static_cast<unsigned>(nbox * g.box * 128) + tb);
        for (int bx = 0; bx < nbox; ++bx)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                    ptx::smem_u32(As(s) + static_cast<size_t>(bx) * g.box * 128)),
                "l"(&tmap), "r"(static_cast<int>(col0)), "r"(static_cast<int>(k0 + g.box * bx)), "r"(ptx::smem_u32(&full[s]))
                : "memory");
        ptx::bulk_g2s(const_cast<uint16_t*>(Ts(s)), g.tiles + (c * g.nrb + rb) * g.blk_stride, tb, &full[s]);
    };
    double acc[4][2][2];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[q][j][0] = acc[q][j][1] = 0.0;
    if (tid == 0)
        for (int s = 0; s < g.ns && cb + s < ce; ++s) issue(cb + s, s);
    const unsigned vhi = static_cast<unsigned>(__double2hiint(g.val)), vlo = static_cast<unsigned>(__double2loint(g.val));
    const unsigned rowkey = 0x2000u | (static_cast<unsigned>(lg) << 10);  // valid | row lg
    const unsigned lgu = static_cast<unsigned>(lg);
    int s = 0;
    unsigned phase = 0;
    for (int64_t c = cb; c < ce; ++c) {
        ptx::mbar_wait(&full[s], phase);
        const unsigned char* Ab = As(s);
        const uint16_t* T = Ts(s);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int tb = warp + 32 * q;
            const int g0 = T[tb], g1 = T[tb + 1];
            const uint16_t* ep = T + kTdHdr + lr;
            for (int gi = g0; gi < g1; gi += 4) {
                const unsigned en = ep[gi];
                // A-fragment: +-val where the entry's row is this lane's row lg
                // (valid bit and row compared in one mask), 0 elsewhere -- built
                // on the high word: sign flip by XOR, zero by AND
                const unsigned hit = ((en & 0x3c00u) == rowkey) ? 0xffffffffu : 0u;
                const unsigned hi = (vhi ^ ((en & 0x8000u) << 16)) & hit;
                const double a = __hiloint2double(static_cast<int>(hi), static_cast<int>(vlo & hit));
                // B-fragments: column tile 0 = the slab's even columns, tile 1 =
                // its odd columns, so lane lg's two operands (columns 2lg and
                // 2lg + 1 of row k) are one 16-byte unit: unit lg ^ (k & 7) of
                // the 128-byte-swizzled row, one LDS.128 for both DMMAs
                const unsigned k = en & 1023u;
                const double2 bb = *reinterpret_cast<const double2*>(Ab + ((k << 7) | (((lgu ^ k) & 7u) << 4)));
                dmma_f64(acc[q][0][0], acc[q][0][1], a, bb.x);
                dmma_f64(acc[q][1][0], acc[q][1][1], a, bb.y);
            }
        }
        // no block barrier: the last warp done with stage s refills it with
        // chunk c + ns, so warps drift up to ns - 1 chunks apart and uneven
        // per-tile group counts average out
        __syncwarp();
        if (lane == 0 && atomicAdd(&done[s], 1) == 31) {
            done[s] = 0;
            if (c + g.ns < ce) issue(c + g.ns, s);
        }
        if (++s == g.ns) {
            s = 0;
            phase ^= 1u;
        }
    }
    double* Y = g.Yw + split * g.ldw * g.d;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t r = static_cast<int64_t>(rb) * kTdRows + (warp + 32 * q) * 8 + lg;
        if (r < g.d)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int64_t col = col0 + 2 * (2 * lr + i) + j;  // tile j holds the columns of parity j
                    if (col < g.ldw) Y[col * g.d + r] = acc[q][j][i];
                }
    }
}

uint64_t lemire_thresh(uint64_t d) { return (0 - d) % d; }

}  // namespace

void generate_sparse_sign_dev(slq_ctx* ctx, int64_t d, int64_t zeta, uint64_t seed,
                              int64_t col_begin, int64_t ncols, uint32_t* compact,
                              int64_t* rows64, double* vals, int64_t* colptr,
                              unsigned long long* stats) {
    if (zeta > d || zeta < 1) fail(SLQ_INVALID_SPARSITY, "generate_sparse_sign: need 1 <= zeta <= d");
    if (ncols <= 0) {
        if (colptr) SLQ_CUDA_CHECK(cudaMemsetAsync(colptr, 0, sizeof(int64_t), ctx->stream));
        return;
    }
    GenArgs a{d, zeta, col_begin, ncols, mix64(seed), lemire_thresh(static_cast<uint64_t>(d)),
              1.0 / std::sqrt(static_cast<double>(zeta)), compact, rows64, vals, colptr, stats};
    const bool warp_path = zeta <= 32 && d < (int64_t(1) << 31);
    if (warp_path) {
        int G = 1;
        while (G < zeta) G <<= 1;
        const int64_t cols_per_block = 8 * (32 / G);
        const unsigned grid = static_cast<unsigned>(ceil_div(ncols, cols_per_block));
        switch (G) {
            case 1: gen_warp_kernel<1><<<grid, 256, 0, ctx->stream>>>(a); break;
            case 2: gen_warp_kernel<2><<<grid, 256, 0, ctx->stream>>>(a); break;
            case 4: gen_warp_kernel<4><<<grid, 256, 0, ctx->stream>>>(a); break;
            case 8: gen_warp_kernel<8><<<grid, 256, 0, ctx->stream>>>(a); break;
            case 16: gen_warp_kernel<16><<<grid, 256, 0, ctx->stream>>>(a); break;
            default: gen_warp_kernel<32><<<grid, 256, 0, ctx->stream>>>(a); break;
        }
        SLQ_LAUNCH_CHECK(ctx);
    } else {
        if (!rows64) fail(SLQ_INVALID_ARG, "generic generator path needs an int64 work array");
        if (compact && d >= (int64_t(1) << 31)) fail(SLQ_UNSUPPORTED, "compact sketch needs d < 2^31");
        const unsigned grid = static_cast<unsigned>(ceil_div(ncols, 128));
        gen_generic_kernel<<<grid, 128, 0, ctx->stream>>>(a);
        SLQ_LAUNCH_CHECK(ctx);
    }
}

namespace {

ChunkPlan plan_chunks(int64_t m, int64_t d, int64_t zeta_max, int W) {
    ChunkPlan p{};
    int zp = 1;
    while (zp < zeta_max) zp <<= 1;
    p.ptr_stride = round_up(d + 1, 8);
    // largest power-of-two K (<= 2048, entries <= 16384 for u16 offsets) whose
    // double-buffered stage (A slab 8*W B/row + row pointers + entries) fits
    // (the sparse path, W = 0, keeps the W = 4 plan: measured at C4, its one-warp
    // counting sort is faster on 1024-row chunks (3.2 ms) than on 2048 (4.8 ms),
    // which the halved S^T row build (1.45 -> 1.1 ms) does not make up)
    const int64_t rowb = 8 * std::max(W, 4);
    int K = 2048;
    while (K > 16 && (static_cast<int64_t>(K) * zp > 16384 ||
                      2 * (K * rowb + p.ptr_stride * 2 + round_up(static_cast<int64_t>(K) * zeta_max, 8) * 2) >
                          220 * 1024))
        K >>= 1;
    p.K = K;
    p.KB = 0;
    while ((1 << p.KB) < p.K) ++p.KB;
    p.cap = 16384;
    p.nchunks = ceil_div(m, p.K);
    p.ent_stride = round_up(static_cast<int64_t>(p.K) * zeta_max, 8);
    return p;
}

// 2D tensor map over the row-major A block (inner dim = ld columns, outer = m
// rows), boxes of 256 rows x W columns, no swizzle (the gather's entries hold
// plain byte offsets k * 8W).
CUtensorMap gather_tensor_map(const double* A, int64_t ld, int64_t m, int W, bool swizzle128 = false,
                              unsigned box_rows = 256) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        SLQ_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) fail(SLQ_CUDA, "cuTensorMapEncodeTiled not available");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (W < 2) return map;  // 1-column slabs stage with cp.async
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(std::max<int64_t>(m, 1))};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(W), box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE,
                              swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SLQ_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return map;
}

template <int RPT, int W, bool EXACT>
void launch_gather_t(slq_ctx* ctx, const GatherArgs& g, int64_t nslabs, size_t smem) {
    auto kern = gather_kernel<RPT, W, EXACT>;
    SLQ_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const CUtensorMap map = gather_tensor_map(g.A, g.ld, g.m, W);
    dim3 grid(static_cast<unsigned>(nslabs), static_cast<unsigned>(g.nsplit));
    kern<<<grid, kGThreads, smem, ctx->stream>>>(map, g);
    SLQ_LAUNCH_CHECK(ctx);
}

// slab width W and rows per thread: y holds RPT x W = 16 doubles per thread
template <bool EXACT>
void launch_gather(slq_ctx* ctx, const GatherArgs& g, int rpt, int W, int64_t nslabs, size_t smem) {
    switch (rpt) {
        case 1: launch_gather_t<1, 4, EXACT>(ctx, g, nslabs, smem); break;
        case 2: launch_gather_t<2, 4, EXACT>(ctx, g, nslabs, smem); break;
        case 4: launch_gather_t<4, 4, EXACT>(ctx, g, nslabs, smem); break;
        case 8: launch_gather_t<8, 2, EXACT>(ctx, g, nslabs, smem); break;   // 4096 < d <= 8192: 2-column slabs
        case 16: launch_gather_t<16, 1, EXACT>(ctx, g, nslabs, smem); break; // d <= 16384: 1-column slabs
        default: fail(SLQ_UNSUPPORTED, "sketch_apply: d > 16384 not supported by the register-slab gather");
    }
    (void)W;
}

}  // namespace

void generate_sparse_rows_dev(slq_ctx* ctx, int64_t n, int64_t nnz, uint64_t seed, int64_t row_begin, int64_t m,
                              const double* scale, int64_t* rowptr, int32_t* colidx, double* vals) {
    if (nnz < 1 || nnz > n) fail(SLQ_INVALID_SPARSITY, "sparse rows: need 1 <= nnz per row <= n");
    DevBuf work;
    int64_t* w = static_cast<int64_t*>(work.ensure(sizeof(int64_t) * std::max<int64_t>(1, m * nnz)));
    sparse_rows_kernel<<<static_cast<unsigned>(ceil_div(m + 1, 128)), 128, 0, ctx->stream>>>(
        n, nnz, mix64(seed), lemire_thresh(static_cast<uint64_t>(n)), row_begin, m, scale, rowptr, colidx, vals, w);
    SLQ_LAUNCH_CHECK(ctx);
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}

static ChunkCsr build_chunk_csr_plan(slq_ctx* ctx, const uint32_t* compact, const int64_t* colptr_dev,
                                     int64_t zeta_max, int64_t m, int64_t d, int gather_width, const ChunkPlan& plan) {
    Workspace& ws = ctx->ws;
    ChunkCsr cc;
    cc.plan = plan;
    const ChunkPlan& cp = cc.plan;
    // slack: row-part slices may run past the last chunk
    cc.ptr = static_cast<uint16_t*>(ws.chunk_ptr.ensure(sizeof(uint16_t) * (cp.ptr_stride * cp.nchunks + d + 64)));
    cc.ent = static_cast<uint16_t*>(ws.chunk_ent.ensure(sizeof(uint16_t) * cp.ent_stride * cp.nchunks));
    cc.flag = static_cast<int*>(ws.flags.ensure(4096));
    SLQ_CUDA_CHECK(cudaMemsetAsync(cc.flag, 0, sizeof(int), ctx->stream));
    BucketArgs ba{compact, colptr_dev, zeta_max, m, d, cp.K, cp.KB, cp.ptr_stride, cp.ent_stride, cc.ptr, cc.ent,
                  cp.cap, cc.flag, gather_width};
    static const bool bitonic = slq_env_flag("SLQ_BUCKET_BITONIC");  // diagnostics: the bitonic network
    if (!colptr_dev && gather_width == 0 && d <= kBcMaxD && !bitonic) {
        const size_t csmem = sizeof(uint16_t) * static_cast<size_t>((d + 7) & ~int64_t(7));
        bucketize_count_kernel<<<static_cast<unsigned>(cp.nchunks), 32, csmem, ctx->stream>>>(ba);
        SLQ_LAUNCH_CHECK(ctx);
        return cc;
    }
    const size_t bsmem = sizeof(uint32_t) * cp.cap;
    SLQ_CUDA_CHECK(cudaFuncSetAttribute(bucketize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(bsmem)));
    bucketize_kernel<<<static_cast<unsigned>(cp.nchunks), 1024, bsmem, ctx->stream>>>(ba);
    SLQ_LAUNCH_CHECK(ctx);
    return cc;
}

ChunkCsr build_chunk_csr(slq_ctx* ctx, const uint32_t* compact, const int64_t* colptr_dev, int64_t zeta_max,
                         int64_t m, int64_t d, int gather_width) {
    return build_chunk_csr_plan(ctx, compact, colptr_dev, zeta_max, m, d, gather_width,
                                plan_chunks(m, d, zeta_max, gather_width));
}

namespace {

// K2d (fast mode, device-resident A): tile gather on the FP64 tensor cores.
// Returns false if a chunk overflowed its bucket (caller falls back to the
// register gather, which has no per-row-block capacity).
bool sketch_apply_dmma(slq_ctx* ctx, const slq_dense* A, int64_t d, const uint32_t* compact,
                       const int64_t* colptr_dev, int64_t zeta_max, double val, double* Y) {
    const int64_t m = A->m, ld = A->ld, ncols_out = A->n + 1;
    int zp = 1;
    while (zp < zeta_max) zp <<= 1;
    ChunkPlan p{};
    // K rows per chunk: 768 (k_local < 1024, 10 bits of a tile entry; 3 TMA
    // boxes) when the chunk's K * zeta entries fit a u16 chunk-CSR, else the
    // largest power of two that does; boxes of min(256, K) rows
    p.K = 768;
    if (static_cast<int64_t>(p.K) * zp > 16384) {
        p.K = 512;
        while (p.K > 16 && static_cast<int64_t>(p.K) * zp > 16384) p.K >>= 1;
    }
    p.KB = 0;
    while ((1 << p.KB) < p.K) ++p.KB;
    p.cap = 16384;
    p.nchunks = ceil_div(m, static_cast<int64_t>(p.K));
    p.ptr_stride = round_up(d + 1, 8);
    p.ent_stride = round_up(static_cast<int64_t>(p.K) * zeta_max, 8);
    const int nrb = static_cast<int>(ceil_div(d, static_cast<int64_t>(kTdRows)));
    const int64_t rows_rb = std::min<int64_t>(kTdRows, d);
    const int64_t expect = static_cast<int64_t>(p.K) * zeta_max * rows_rb / d;
    int64_t cap = round_up(std::min<int64_t>(static_cast<int64_t>(p.K) * zeta_max, 2 * expect + 256) + 3 * kTdTiles, 8);
    if (const char* e = std::getenv("SLQ_TD_CAP")) cap = std::max<int64_t>(8, round_up(std::atoll(e), 8));  // tests: force overflow
    const int64_t blk_stride = kTdHdr + cap;
    Workspace& ws = ctx->ws;
    uint16_t* tiles = static_cast<uint16_t*>(ws.tile_ent.ensure(sizeof(uint16_t) * p.nchunks * nrb * blk_stride));
    int* flags = static_cast<int*>(ws.flags.ensure(4096));
    SLQ_CUDA_CHECK(cudaMemsetAsync(flags, 0, 2 * sizeof(int), ctx->stream));
    const int64_t ntile = ceil_div(d, static_cast<int64_t>(8));
    if (!colptr_dev && ntile <= kTbMaxTiles) {
        // uniform zeta: one fused pass from the generator's entries to the tile layout
        TileBucketArgs ta{compact, zeta_max, m, d, p.K, nrb, static_cast<int>(cap), blk_stride, tiles, flags + 1};
        const int64_t nhp = (ntile + 1) / 2;
        const size_t tsmem = sizeof(int) * (32 * nhp + 2 * ntile + nrb);
        SLQ_CUDA_CHECK(cudaFuncSetAttribute(tile_bucketize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(tsmem)));
        tile_bucketize_kernel<<<static_cast<unsigned>(p.nchunks), 1024, tsmem, ctx->stream>>>(ta);
        SLQ_LAUNCH_CHECK(ctx);
    } else {
        ChunkCsr cc = build_chunk_csr_plan(ctx, compact, colptr_dev, zeta_max, m, d, 0, p);
        RepackArgs ra{cc.ptr, cc.ent, p.ptr_stride, p.ent_stride, d, nrb, static_cast<int>(cap), blk_stride, tiles,
                      flags + 1};
        tile_repack_kernel<<<static_cast<unsigned>(p.nchunks), 1024, 0, ctx->stream>>>(ra);
        SLQ_LAUNCH_CHECK(ctx);
    }

    const int64_t ldw = round_up(ncols_out, 16);
    const int64_t nslabs = ldw / 16;
    const size_t a_bytes = static_cast<size_t>(p.K) * 128;
    const size_t t_bytes = round_up(static_cast<int64_t>(blk_stride) * 2, 1024);
    const size_t st = a_bytes + t_bytes;
    const int ns = static_cast<int>(std::min<size_t>(kTdMaxStages, (226 * 1024 - 1024) / st));
    if (ns < 2) return false;
    const size_t smem = ns * st + 1024;
    int64_t nsplit = 1;
    {
        double best = 1e30;
        const int64_t ctas = nslabs * nrb;
        for (int64_t s = 1; s <= 16 && s <= p.nchunks; ++s) {
            const double waves = std::ceil(static_cast<double>(ctas * s) / ctx->num_sms);
            const double cost = waves / s + 0.02 * s;
            if (cost < best - 1e-9) {
                best = cost;
                nsplit = s;
            }
        }
    }
    double* Yw = (nsplit == 1 && ldw == ncols_out) ? Y
                 : static_cast<double*>(ws.ypart.ensure(sizeof(double) * nsplit * ldw * d));
    const int box = std::min(256, p.K);
    TdArgs g{m, d, ldw, p.K, box, nsplit, 0, p.nchunks, tiles, blk_stride, nrb, ns, val, Yw};
    SLQ_CUDA_CHECK(cudaFuncSetAttribute(gather_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    const CUtensorMap map = gather_tensor_map(A->A, ld, m, 16, true, static_cast<unsigned>(box));
    gather_dmma_kernel<<<dim3(static_cast<unsigned>(nrb), static_cast<unsigned>(nslabs), static_cast<unsigned>(nsplit)),
                         1024, smem, ctx->stream>>>(map, g);
    SLQ_LAUNCH_CHECK(ctx);
    if (ctx->defer_status) {
        // inside a solve: an overflow (never seen at the shipped capacities) is
        // recorded on the device and the solve is redone with the register gather
        defer_status_dev(ctx, flags, kCondAny2, kStatusSketchOverflow);
    } else {
        int hflag[2] = {0, 0};
        SLQ_CUDA_CHECK(cudaMemcpyAsync(hflag, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (hflag[0] || hflag[1]) return false;
    }
    if (Yw != Y) {
        if (nsplit == 1) {
            SLQ_CUDA_CHECK(cudaMemcpyAsync(Y, Yw, sizeof(double) * d * ncols_out, cudaMemcpyDeviceToDevice, ctx->stream));
        } else {
            const int64_t tot = d * ncols_out;
            reduce_splits_kernel<<<static_cast<unsigned>(ceil_div(tot, 256)), 256, 0, ctx->stream>>>(Yw, nsplit, d, ldw,
                                                                                                    ncols_out, Y);
            SLQ_LAUNCH_CHECK(ctx);
        }
    }
    return true;
}

}  // namespace

void check_chunk_csr(slq_ctx* ctx, const ChunkCsr& cc) {
    if (ctx->defer_status) {  // inside a solve: checked once at the end
        defer_status_dev(ctx, cc.flag, kCondNonzero, SLQ_UNSUPPORTED);
        return;
    }
    int hflag = 0;
    SLQ_CUDA_CHECK(cudaMemcpyAsync(&hflag, cc.flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SLQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (hflag) fail(SLQ_UNSUPPORTED, "sketch_apply: a chunk exceeded 16384 sketch entries");
}

DenseGather dense_gather_plan(slq_ctx* ctx, int64_t m, int64_t n, int64_t ld, int64_t d, const uint32_t* compact,
                              const int64_t* colptr_dev, int64_t zeta, double val, bool exact, double* Y,
                              bool incremental) {
    if (d > 16384) fail(SLQ_UNSUPPORTED, "sketch_apply: d > 16384 not supported");
    if (d >= (int64_t(1) << 21)) fail(SLQ_UNSUPPORTED, "sketch_apply: d too large for chunk keys");
    Workspace& ws = ctx->ws;
    DenseGather G;
    G.m = m;
    G.d = d;
    G.ld = ld;
    G.ncols_out = n + 1;
    G.val = val;
    G.exact = exact;
    G.Y = Y;
    // W-column slab per CTA, all d rows of the slab in registers (32 doubles per
    // thread: W = 4 up to d = 4096, W = 2 up to 8192, W = 1 up to 16384)
    G.rpt = 1;
    while (G.rpt * kGThreads < d) G.rpt <<= 1;
    G.W = G.rpt <= 4 ? 4 : (G.rpt == 8 ? 2 : 1);
    G.cc = build_chunk_csr(ctx, compact, colptr_dev, zeta, std::max<int64_t>(m, 1), d, G.W);
    const ChunkPlan& cp = G.cc.plan;
    G.ldw = round_up(ld, G.W);
    G.nslabs = G.ldw / G.W;
    // splits along m: balance waves over the SMs unless the exact serial order
    // (or incremental row ranges) is asked for
    G.nsplit = 1;
    if (!exact && !incremental) {
        double best = 1e30;
        for (int64_t s = 1; s <= 16; ++s) {
            if (s > cp.nchunks) break;
            const int64_t ctas = G.nslabs * s;
            const double waves = std::ceil(static_cast<double>(ctas) / ctx->num_sms);
            const double cost = waves / s + 0.02 * s;  // per-split overhead (partials + reduce)
            if (cost < best - 1e-9) {
                best = cost;
                G.nsplit = s;
            }
        }
    }
    G.Yw = (G.nsplit == 1 && G.ldw == G.ncols_out) ? Y
           : static_cast<double*>(ws.ypart.ensure(sizeof(double) * G.nsplit * G.ldw * d));
    G.smem = 2 * round_up(static_cast<int64_t>(cp.K) * G.W * sizeof(double) + cp.ptr_stride * sizeof(uint16_t) +
                              cp.ent_stride * sizeof(uint16_t), 128);
    if (G.smem > 227 * 1024) fail(SLQ_UNSUPPORTED, "sketch_apply: stage exceeds shared memory");
    return G;
}

void dense_gather_rows(slq_ctx* ctx, const DenseGather& G, const double* A, int64_t row_lo, int64_t row_hi) {
    const ChunkPlan& cp = G.cc.plan;
    const int64_t c_lo = row_lo / cp.K, c_hi = std::min(cp.nchunks, ceil_div(row_hi, static_cast<int64_t>(cp.K)));
    if (c_hi <= c_lo) return;
    if (row_lo % cp.K != 0 || (row_hi % cp.K != 0 && row_hi != G.m))
        fail(SLQ_INVALID_ARG, "sketch_apply: row range not aligned to the chunk size");
    GatherArgs g{A, G.ld, G.m, G.d, cp.K, cp.nchunks, G.nsplit, cp.ptr_stride, cp.ent_stride, G.cc.ptr, G.cc.ent,
                 G.val, G.ldw, G.Yw, c_lo, c_hi, c_lo > 0 ? 1 : 0};
    if (G.exact) launch_gather<true>(ctx, g, G.rpt, G.W, G.nslabs, G.smem);
    else launch_gather<false>(ctx, g, G.rpt, G.W, G.nslabs, G.smem);
}

void dense_gather_finish(slq_ctx* ctx, const DenseGather& G) {
    if (G.m == 0) {
        SLQ_CUDA_CHECK(cudaMemsetAsync(G.Y, 0, sizeof(double) * G.d * G.ncols_out, ctx->stream));
    } else if (G.Yw != G.Y) {
        if (G.nsplit == 1) {  // same column-major layout: the first n+1 columns are contiguous
            SLQ_CUDA_CHECK(cudaMemcpyAsync(G.Y, G.Yw, sizeof(double) * G.d * G.ncols_out, cudaMemcpyDeviceToDevice,
                                           ctx->stream));
        } else {
            const int64_t tot = G.d * G.ncols_out;
            reduce_splits_kernel<<<static_cast<unsigned>(ceil_div(tot, 256)), 256, 0, ctx->stream>>>(
                G.Yw, G.nsplit, G.d, G.ldw, G.ncols_out, G.Y);
            SLQ_LAUNCH_CHECK(ctx);
        }
    }
    check_chunk_csr(ctx, G.cc);
}

void sketch_apply_compact_dev(slq_ctx* ctx, const slq_dense* A, int64_t d, const uint32_t* compact,
                              const int64_t* colptr_dev, int64_t zeta, double val, bool exact,
                              double* Y) {
    const int64_t m = A->m;
    if (m == 0) {
        SLQ_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(double) * d * (A->n + 1), ctx->stream));
        return;
    }
    // fast mode: the DMMA tile gather (falls back if a bucket overflowed),
    // except where the register gather measured faster (tools/diag_k2d.py at
    // m = 1e6, n = 500: zeta >= 16 with d <= 2048 -- many entries per row per
    // chunk keep its lanes busy; zeta <= 2 with d >= 2048 -- too little work
    // per A row to repay the tile gather's per-row-block restaging)
    const bool row_gather = slq_env_flag("SLQ_ROW_GATHER") ||  // diagnostics: register gather in fast mode
                            ctx->force_row_gather || (zeta >= 16 && d <= 2048) || (zeta <= 2 && d >= 2048);
    if (!exact && !row_gather && sketch_apply_dmma(ctx, A, d, compact, colptr_dev, zeta, val, Y)) return;
    DenseGather G = dense_gather_plan(ctx, m, A->n, A->ld, d, compact, colptr_dev, zeta, val, exact, Y, false);
    dense_gather_rows(ctx, G, A->A, 0, m);
    dense_gather_finish(ctx, G);
}

void sketch_apply_dev(slq_ctx* ctx, const slq_dense* A, int64_t d, int64_t zeta, uint64_t seed,
                      bool exact, double* Y) {
    if (zeta > d || zeta < 1) fail(SLQ_INVALID_SPARSITY, "apply: need 1 <= zeta <= d");
    if (zeta > 1024) fail(SLQ_UNSUPPORTED, "sketch_apply: zeta > 1024");
    Workspace& ws = ctx->ws;
    const int64_t m = A->m;
    uint32_t* compact = static_cast<uint32_t*>(ws.compact.ensure(sizeof(uint32_t) * std::max<int64_t>(1, m * zeta)));
    int64_t* work = nullptr;
    if (zeta > 32) work = static_cast<int64_t*>(ws.tmp.ensure(sizeof(int64_t) * m * zeta));
    generate_sparse_sign_dev(ctx, d, zeta, seed, A->row_begin, m, compact, work, nullptr, nullptr, nullptr);
    sketch_apply_compact_dev(ctx, A, d, compact, nullptr, zeta, 1.0 / std::sqrt(static_cast<double>(zeta)),
                             exact, Y);
}

}  // namespace slq
