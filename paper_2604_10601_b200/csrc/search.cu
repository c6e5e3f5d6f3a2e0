// search.cu -- gm_count / gm_enumerate: the fine-grained DFS extension of partial matches.
//
// PAPER.md §4-§5 (lines 362-544) re-designed for sm_100a:
//
//  * Initialization phase (§4.3; Alg. 2 line 1): breadth-first expansion of
//    the root candidates level by level (k_expand, one warp per partial match, count pass
//    then write pass) until the pool holds >= tau partial matches.  The pool is stored
//    level-major (pool[i * P + k] = M_k[phi[i]]) so a warp loads 32 pool items with
//    coalesced 128-byte reads.
//  * Fine-grained execution (§4.1) + warp-level batch exploration (§4.2) (k_dfs): each
//    warp owns an execution stack S[level][lane] in shared memory (Alg. 2 §5.1: fields
//    v, pid, and the local candidate set C, kept here as a (begin, length, source-level)
//    slice of the label-partitioned CSR), i.e. O(|V(Q)| * 32) entries independent of
//    d_max (§5.2).  Each round, the 32 lanes take the next 32 tasks T_M(u, v) from the
//    virtual task pool formed by ALL parent lanes' remaining candidate slices (the two
//    cursors of §4.2 / ScatterTask), computed warp-parallel with a shuffle scan instead
//    of Alg. 2's serial leader loop; every lane validates its task (candidate filter bit,
//    injectivity and backward-neighbour adjacency by binary search, fused in one walk up
//    the pid chain, §5.2 "We fuse these checks into a single loop"); a ballot decides
//    whether to descend (Alg. 2 lines 15-16).
//  * Load balancing (§4.3): warps fetch 32 pool items at a time with one atomicAdd (the
//    pool items become the 32 lanes of the base level: batch exploration starts at the
//    pool); an idle warp posts one steal request (global counter); a busy warp that
//    claims a request hands off the untouched part of its shallowest splittable stack
//    level (its last untouched parent lane, or the upper half of the current slice)
//    through a bounded MPMC ring -- the paper's "idle warps receive half of the work
//    from busy warps by splitting the execution stack", via a ring instead of a direct
//    warp-to-warp hand-off.  Termination: `work` counts warps holding work plus items in
//    the ring; a warp exits when the pool is exhausted and work == 0.
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <vector>

#include "gm_internal.cuh"

namespace gm {

constexpr uint32_t FULL = 0xffffffffu;
// per-warp scratch rows (32 words each) after the WarpStack: rows_chk rows of check images,
// then rows_last rows of set/pair-counting words
#define CHK(k, x) scr[(k) * 32u + (x)]
#define LASTW(k, x) scr[(P.rows_chk + (k)) * 32u + (x)]
#define GENW(k, x) scr[(P.rows_chk + P.rows_last + (k)) * 32u + (x)]   // gen_prep's cached slice
// then rows_aux rows of per-lane counting state (set / pair counting kernels only):
// 0 lastmb, 1 lastlb, 2 lastub (prep_last / prep_two), 3 tacc (pair counting)
#define AUXW(k, x) scr[(P.aux_row + (k)) * 32u + (x)]
#ifndef GM_CHK_ORDER
#define GM_CHK_ORDER 1
#endif
#ifndef GM_CHK_HUBFIRST
#define GM_CHK_HUBFIRST 0
#endif
#ifndef GM_VHUB
#define GM_VHUB 1
#endif
#ifndef GM_DFS_MINB
#define GM_DFS_MINB 9      // resident 128-thread blocks per SM for the 8-level kernel (<= 56 registers)
#endif
// 16/24/32-level kernels: shared memory (the stack, 6-15 KB per warp) limits their residency,
// so they are compiled for blocks of up to GM_WPB_WIDE warps at 72 registers (28 warps per
// SM), and the host picks, per query, the block size that keeps the most warps resident
#ifndef GM_WPB_WIDE
#define GM_WPB_WIDE 14
#endif
#ifndef GM_MINB16
#define GM_MINB16 (28 / GM_WPB_WIDE)
#endif
#ifndef GM_MINB32
#define GM_MINB32 (28 / GM_WPB_WIDE)
#endif
#define GM_DFS_MINB_D(D) ((D) <= 8 ? GM_DFS_MINB : ((D) <= 16 ? GM_MINB16 : GM_MINB32))
#ifndef GM_TWO_STAGE
#define GM_TWO_STAGE 0     // pair-count intersection: stage a short non-hub longer list in shared
#endif                     // memory with cp.async.bulk (TMA) and search it there
#if GM_TWO_STAGE
constexpr uint32_t kStageWords = 256;          // staging buffer: 8 scratch rows per warp
#endif
#ifndef GM_WIDE
#define GM_WIDE 1          // two tasks per lane per round at the terminal per-parent level
#endif
#ifndef GM_WIDE_MIN_D
#define GM_WIDE_MIN_D 8    // ... in the kernels with at least this many stack levels
#endif
#ifndef GM_WIDE_T
#define GM_WIDE_T 2        // tasks per lane in a wide round (4: 12-30 % slower on rmat18/24)
#endif
#ifndef GM_WIDE_TSIB
#define GM_WIDE_TSIB 2     // ... in the 8-level sibling-prefix kernel (short prefix slices, one probe each)
#endif
#ifndef GM_WIDE_T16
#define GM_WIDE_T16 2      // ... in the 16-level kernel
#endif
#ifndef GM_WIDE_LOOP8
#define GM_WIDE_LOOP8 0    // wide rounds' per-task counting in a loop (1) or unrolled (0): 8-level kernel
#endif
#ifndef GM_WIDE_LOOP16
#define GM_WIDE_LOOP16 1   // ... 16/24/32-level kernels
#endif
#define GM_WIDE_LOOP_D(D) ((D) <= 8 ? GM_WIDE_LOOP8 : GM_WIDE_LOOP16)
#ifndef GM_WIDE_PAIR
#define GM_WIDE_PAIR 1     // wide rounds also at the pair-counting level (leaves of different labels)
#endif
#ifndef GM_WIDE_T32
#define GM_WIDE_T32 4      // ... in the 32-level kernel (4 vs 2: rmat26 +4 to +23 % tasks/s)
#endif
#ifndef GM_HUB_SUMMARY
#define GM_HUB_SUMMARY 0   // 1: the kernels use the hub index's summary level when the graph has one
#endif                     // (0: the test is compiled out -- rmat24 +17-19 %, rmat26 +3-52 % tasks/s)
#ifndef GM_TWO_VEC8
#define GM_TWO_VEC8 0      // ... and 256-element rounds (two 16-byte loads, 8 probes per lane)
#endif
#ifndef GM_TWO_VEC
#define GM_TWO_VEC 1       // pair-counting intersection: 128-element rounds with 16-byte loads
#endif
#ifndef GM_PROBES_WIDE
#define GM_PROBES_WIDE 1   // checks per pass in the 16/32-level kernels (process()): on rmat24 1 beat
#endif                     // 2 by 3-15 % and 4 lost 13-51 % tasks/s (wasted DRAM probes)
#ifndef GM_WORDS
#define GM_WORDS 1         // count algorithmic words (gm_run_stats.words); 0 compiles the counting out
#endif
#if GM_WORDS
#define GM_ADD_WORDS(x) (WORDS ? (void)(my_words += (x)) : (void)0)
#else
#define GM_ADD_WORDS(x) ((void)0)
#endif
#ifndef GM_D24
#define GM_D24 1           // a 24-level count kernel for 17-24-vertex queries
#endif
#ifndef GM_SIB
#define GM_SIB 1           // sibling prefixes for clique-like last levels (sib_append)
#endif
#ifndef GM_GEN_CACHE
#define GM_GEN_CACHE 1     // GenerateTask at the hot level with a per-grandparent cached part (gen_prep)
#endif
#ifndef GM_PREFETCH_ROWS
#define GM_PREFETCH_ROWS 0 // prefetch the task vertex's row offsets for the counting step (A/B)
#endif
#ifndef GM_TEAM_CODE
#define GM_TEAM_CODE 1     // (A/B switch) 0 compiles the cross-GPU stealing team code out of the kernels
#endif
#define GM_TEAMN(P) (GM_TEAM_CODE ? (P).team_n : 0u)
#ifndef GM_PACK_PID
#define GM_PACK_PID 1      // 16/24/32-level kernels: the parent lane in the top 5 bits of the vertex word
#endif
#ifndef GM_PACK_CS
#define GM_PACK_CS 1       // the slice's source level in the top 5 bits of its length (416-byte levels)
#endif
#ifndef GM_CUT_MIN
#define GM_CUT_MIN 0       // GenerateTask under symmetry-breaking bounds: the backward row with the
#endif                     // fewest candidates INSIDE the bounds (else: the shortest row, then cut)
constexpr uint32_t kDfsMaxWarps = GM_WPB_WIDE > 4 ? GM_WPB_WIDE : 4;   // largest k_dfs block, any D
// warps per block k_dfs<D> is compiled for (__launch_bounds__): 4 for the register-limited
// 8-level kernels, GM_WPB_WIDE for the shared-memory-limited deeper ones
template <int D>
constexpr uint32_t dfs_max_warps() { return D <= 8 ? 4u : (uint32_t)GM_WPB_WIDE; }
constexpr uint32_t kItemWords = 6 + kMaxQ;     // [depth, cb, cl, cs, home, epoch, prefix[kMaxQ]]
constexpr uint32_t kMaxTeam = 8;               // ranks of a stealing team (gm_team)
constexpr int kModePlain = 0, kModeSet = 1, kModePair = 2, kModePat = 3;   // k_dfs MODE
constexpr uint32_t kSibCs = GM_PACK_CS ? 31u : 0xffu;   // source level of a slice in the sibling buffer
constexpr uint32_t kSibCap = 256;              // sibling-prefix entries per parent lane

// Global control block.  Every field that many warps poll or update lives on its own
// 128-byte line so that the pollers of one do not serialise the atomics of another.
struct Ctrl {
    alignas(128) unsigned long long pool_ctr;
    alignas(128) int work;                    // warps holding work + items in the ring
    alignas(128) int requests;                // posted steal requests not yet served
    alignas(128) unsigned long long q_head;   // ring positions (monotone, 64-bit: never wrap)
    alignas(128) unsigned long long q_tail;
    alignas(128) int abort;
    alignas(128) unsigned long long tword;    // team: (epoch << 32) | lineage work count
    unsigned long long t0;                    // globaltimer at the first warp's start
    alignas(128) unsigned long long out_ctr;
    alignas(128) unsigned long long count;
    int overflow;               // the count wrapped past 2^64 - 1
    unsigned long long tasks;
    unsigned long long rounds;
    unsigned long long words;   // algorithmic 4-byte words read by k_dfs
    unsigned long long donations;
};

#ifdef GM_LEVEL_STATS
__device__ unsigned long long g_level_tasks[32], g_level_pass[32];   // debug build: tasks / passes per level
#endif

struct SearchParams {
    const uint32_t *__restrict__ offs;
    const uint32_t *__restrict__ nbr;
    const uint32_t *__restrict__ cand;
    uint32_t S, nq, words, use_cand;
    uint32_t lab[kMaxQ];        // L(phi[l])
    uint32_t bw[kMaxQ];         // backward positions of phi[l]
    uint32_t candoff[kMaxQ];    // word offset of phi[l]'s candidate bitmap (phi[l] * words)
    uint32_t cand_needed;       // bit l: the filter of phi[l] is not implied by its backward edges
    uint32_t same_lab[kMaxQ];   // bit i of same_lab[l]: i < l and L(phi[i]) == L(phi[l])
    uint32_t sb_gt[kMaxQ];      // symmetry breaking: bit i of sb_gt[l]: M[phi[l]] > M[phi[i]] required
    uint32_t sb_lt[kMaxQ];      //                    bit i of sb_lt[l]: M[phi[l]] < M[phi[i]] required
    uint32_t walk_low[kMaxQ];   // lowest level process() must visit at level l (l if none)
    uint32_t col[kMaxQ];        // output column of position l (= phi[l])
    const uint32_t *pool;       // level-major, pool_size items of depth d0
    unsigned long long pool_size;
    uint32_t d0;
    uint32_t steal;
    Ctrl *ctrl;
    uint32_t batch;             // pool items fetched per warp (<= 32)
    unsigned long long *pool_ctr;  // &ctrl->pool_ctr, or a counter shared across ranks
    uint32_t pool_sys;          // 1: pool_ctr is shared by several GPUs (system-scope atomics)
    uint32_t *q_items;          // q_cap * kItemWords
    unsigned long long *q_seq;  // q_cap per-slot sequence numbers (Vyukov bounded MPMC ring)
    unsigned long long q_cap;
    const uint32_t *__restrict__ hub_bits;  // hub bitmaps (row w for device ids w < nhubs)
    const uint32_t *__restrict__ hub_summ;  // summary rows (1 bit per 256 vertices), or NULL
    uint32_t summ_words, summ_first;        // hubs h >= summ_first have row h - summ_first
    uint32_t nhubs;                         // 0: no hub index
    uint32_t hub_words;
    const uint32_t *__restrict__ new2old;   // device id -> original id (enumerate output)
    const uint32_t *__restrict__ old2new;   // original id -> device id (user roots)
    uint32_t bulk_last;         // 1: count the last level by set counting (count_last)
    uint32_t last_b;            // position of phi[last]'s single backward neighbour
    uint32_t last_same;         // positions i < last, i != last_b, with L(phi[i]) == L(phi[last])
    uint32_t last_adj;          // positions adjacent to phi[last_b] in Q
    uint32_t last_low;          // deepest level prep_last must visit
    uint32_t last_k;            // popc(last_same & ~last_adj & below last-1): parked images per parent
    uint32_t last_ka;           // with last_sb: popc(last_same & last_adj & below last-1), parked after
    uint32_t last_sb;           // 1: phi[last] carries symmetry-breaking bounds
    uint32_t bulk_two;          // 1: count the last TWO levels per partial match (count_two)
    uint32_t two_b6, two_b7;    // positions of the single backward neighbours of phi[last-1], phi[last]
    uint32_t two_same6, two_same7;  // positions i <= last-2 (i != b) labelled like phi[last-1] / phi[last]
    uint32_t two_adj6, two_adj7;    // ... whose query vertex is adjacent to phi[b6] / phi[b7]
    uint32_t two_low;           // deepest level count_two's walk visits
    uint32_t two_walk;          // 1: a per-task row (b6 or b7 == last-2) has same-label images below
    uint32_t two_stage_row;     // GM_TWO_STAGE: first rows_last row of the staging buffer
    uint32_t rows_chk;          // scratch rows for check images (max checks of a task / par-level list)
    uint32_t rows_last;         // scratch rows for set/pair-counting words
    uint32_t gen_level;         // GenerateTask of this level uses gen_prep's per-grandparent slice (0: off)
    uint32_t rows_gen;          // scratch rows for it (5 or 0)
    uint32_t warp_stride;       // bytes of shared memory per warp: WarpStack + scratch rows
    uint32_t levels;            // stack levels allocated per warp (WarpStack.lv[0 .. levels))
    uint32_t rows_aux;          // scratch rows of counting state (AUXW): 3 set counting, 4 pair, else 0
    uint32_t aux_row;           // their first row: rows_chk + rows_last + rows_gen
    uint32_t stack_bytes;       // header + levels * sizeof(StackLevel): the scratch rows start there
    uint32_t par_level;         // level whose checks are kept per parent (prep_checks), or ~0u
    uint32_t par_low;           // deepest level prep_checks visits
    uint32_t *out;              // enumerate rows (nq words each)
    unsigned long long out_cap;
    uint32_t stop_at_cap;       // enumerate: stop once out_cap rows are written
    // cross-GPU stealing (gm_team): every rank's control block and steal ring mapped through
    // peer memory; team_n = 0 when this launch steals only within its GPU.  A unit of work is
    // counted in the `work` word of its lineage rank (`home`: the rank whose pool batch it
    // came from), wherever it runs, so a rank's count, once zero with the pool exhausted,
    // stays zero and the team terminates when every rank's count reads zero.
    uint32_t team_n, team_rank, epoch;      // epoch: this search's number in the team's sequence
    Ctrl *team_ctrl[kMaxTeam];
    uint32_t *team_items[kMaxTeam];
    unsigned long long *team_seq[kMaxTeam];
    uint32_t no_pool;           // GM_FLAG_NO_POOL (diagnostic): take no pool batches, only steal
    // sibling prefixes: candidates of phi[sib_level] taken from the valid
    // candidates of phi[sib_level - 1] under the same parent that precede the task's own vertex
    uint32_t *sib;              // per warp: 32 parent lanes x sib_cap recorded siblings, or NULL
    uint32_t sib_level;         // 0: off
    uint32_t sib_cap;           // siblings recorded per parent (later ones use the normal slice)
    uint32_t sib_chk;           // positions phi[sib_level] must still be checked against: bw \ bw(sib_level-1)
    unsigned long long limit_ns;     // time limit of this launch (0 = none)
};

// ------------------------------------------------------------------ device helpers

__device__ __forceinline__ uint32_t ld_nc(const uint32_t *p) { return __ldg(p); }

// v in sorted nbr[lo, hi)?  Branch-free lower bound; ceil(log2(hi-lo)) + 1 word reads,
// added to `words` (the algorithmic-bytes counter).
__device__ __forceinline__ bool contains(const uint32_t *__restrict__ nbr, uint32_t lo, uint32_t hi, uint32_t v,
                                         uint32_t &words) {
    uint32_t n = hi - lo;
    if (n == 0) return false;
    const uint32_t *base = nbr + lo;
    while (n > 1) {
        const uint32_t half = n >> 1;
        base = (ld_nc(base + half) <= v) ? base + half : base;
        n -= half;
        ++words;
    }
    ++words;
    return ld_nc(base) == v;
}

// Index of the first element >= x in the sorted a[0..n) (n if none).
__device__ __forceinline__ uint32_t lower_bound_idx(const uint32_t *__restrict__ a, uint32_t n, uint32_t x,
                                                    uint32_t &words) {
    uint32_t lo = 0;
    while (n > 0) {
        const uint32_t half = n >> 1;
        ++words;
        if (ld_nc(a + lo + half) < x) { lo += half + 1; n -= half + 1; }
        else n = half;
    }
    return lo;
}

__device__ __forceinline__ bool cand_bit(const SearchParams &P, uint32_t l, uint32_t v, uint32_t &words) {
    if (!P.use_cand) return true;
    ++words;
    return (ld_nc(P.cand + P.candoff[l] + (v >> 5)) >> (v & 31)) & 1u;
}

// Summary bit of hub h for vertex x: 0 means no neighbour of h in x's 256-vertex block
// (so x is not one); always 1 without a summary level.
// SUMM = false compiles the summary level out: the L2-resident 8-level kernel (small graphs,
// no summary by default) keeps its register budget; ignoring a summary is always correct
// (the bitmaps are complete), it only forgoes the shortcut.
template <bool SUMM = true>
__device__ __forceinline__ uint32_t hub_summ_word(const SearchParams &P, uint32_t h, uint32_t x, uint32_t &words) {
#if GM_HUB_SUMMARY
    if (SUMM && P.hub_summ && h >= P.summ_first) {
        ++words;
        return ld_nc(P.hub_summ + (unsigned long long)(h - P.summ_first) * P.summ_words + (x >> 13));
    }
#endif
    return 0xffffffffu;
}
__device__ __forceinline__ bool summ_says(uint32_t sw, uint32_t x) { return (sw >> ((x >> 8) & 31)) & 1u; }

// x in N(h) for a hub h: the summary word (if any), then the bitmap word
template <bool SUMM = true>
__device__ __forceinline__ bool hub_bit(const SearchParams &P, uint32_t h, uint32_t x, uint32_t &words) {
    if (!summ_says(hub_summ_word<SUMM>(P, h, x, words), x)) return false;
    ++words;
    return (ld_nc(P.hub_bits + (unsigned long long)h * P.hub_words + (x >> 5)) >> (x & 31)) & 1u;
}

// Is {a, b} an edge?  la = L(a), lb = L(b).  The test is symmetric (b in N_lb(a) iff a in
// N_la(b)), so it takes the cheapest side: the hub bitmap of a or of b if either is a hub
// (device ids are ordered by degree: "is a hub" is w < nhubs), else a binary search of the
// row of the LOWER-degree vertex (the larger device id), which is the shorter list.
template <bool SUMM = true>
__device__ __forceinline__ bool has_edge(const SearchParams &P, uint32_t a, uint32_t la, uint32_t b, uint32_t lb,
                                         uint32_t &words) {
    if (a < P.nhubs || b < P.nhubs) {
        const uint32_t h = a < P.nhubs ? a : b, x = a < P.nhubs ? b : a;
        return hub_bit<SUMM>(P, h, x, words);
    }
    const uint32_t r = a > b ? a : b, x = a > b ? b : a, lx = a > b ? lb : la;
    const uint32_t row = r * P.S + lx;
    words += 2;
    return contains(P.nbr, ld_nc(P.offs + row), ld_nc(P.offs + row + 1), x, words);
}

// acc += x, recording a wrap past 2^64 - 1 in ovf (per-task counts reach |V| * B in pair
// counting, so a lane's running sum can wrap long before the final atomicAdd)
__device__ __forceinline__ void add_count(unsigned long long &acc, unsigned long long x, bool &ovf) {
    const unsigned long long s = acc + x;
    ovf |= s < acc;
    acc = s;
}

// The pool counter.  Shared by several GPUs (peer memory over NVLink, gm_pool_counter_*), a
// device-scope atomic is atomic only among the threads of ONE GPU (PTX memory model), so the
// claim is a system-scope atomicAdd and the poll a relaxed system-scope load; the pool items
// themselves are per-GPU replicas, so no ordering beyond the counter's own atomicity is needed.
__device__ __forceinline__ unsigned long long pool_peek(const SearchParams &P) {
    unsigned long long x;
    if (P.pool_sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(P.pool_ctr) : "memory");
    else x = *(volatile unsigned long long *)P.pool_ctr;
    return x;
}
__device__ __forceinline__ unsigned long long pool_claim(const SearchParams &P, unsigned long long n) {
    return P.pool_sys ? atomicAdd_system(P.pool_ctr, n) : atomicAdd(P.pool_ctr, n);
}

// Scope-dependent atomics of the steal protocol: a team's counters and rings are touched by
// several GPUs, so they take system-scope atomics and loads; alone, device scope.
__device__ __forceinline__ int ld_sys(const int *p) {
    int x;
    asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
    return x;
}
__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long *p) {
    unsigned long long x;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
    return x;
}
__device__ __forceinline__ unsigned long long ld_sys64(const unsigned long long *p) {
    unsigned long long x;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
    return x;
}
// Team counts live in the low half of (epoch << 32) | count: a rank's word tagged with another
// epoch holds no unit of this search (the rank has not started it, or has finished it, which
// needs its lineage count at zero), so consecutive searches need no barrier between them.
__device__ __forceinline__ void work_add(const SearchParams &P, Ctrl *C, uint32_t home, int delta) {
    if (GM_TEAMN(P)) atomicAdd_system(&P.team_ctrl[home]->tword, (unsigned long long)(long long)delta);
    else atomicAdd(&C->work, delta);
}
__device__ __forceinline__ int req_add(const SearchParams &P, Ctrl *C, int delta) {
    return GM_TEAMN(P) ? atomicAdd_system(&C->requests, delta) : atomicAdd(&C->requests, delta);
}
// every rank's lineage count is zero (the whole team is out of work)
__device__ __forceinline__ bool team_idle(const SearchParams &P, volatile Ctrl *VC) {
    if (!GM_TEAMN(P)) return VC->work == 0;
    for (uint32_t r = 0; r < GM_TEAMN(P); ++r) {
        const unsigned long long w = ld_sys64(&P.team_ctrl[r]->tword);
        if ((uint32_t)(w >> 32) == P.epoch && (uint32_t)w != 0) return false;
    }
    return true;
}
// Pop one item from rank r's ring (r = this rank: its own ring); returns its position or ~0.
__device__ __forceinline__ unsigned long long ring_pop(const SearchParams &P, Ctrl *C, uint32_t r) {
    if (!GM_TEAMN(P)) {
        volatile Ctrl *VC = C;
        const unsigned long long pos = VC->q_head;
        const unsigned long long seq = ((volatile unsigned long long *)P.q_seq)[pos % P.q_cap];
        return (seq == pos + 1 && atomicCAS(&C->q_head, pos, pos + 1) == pos) ? pos : ~0ull;
    }
    Ctrl *RC = P.team_ctrl[r];
    const unsigned long long pos = ld_acq_sys(&RC->q_head);
    const unsigned long long seq = ld_acq_sys(P.team_seq[r] + pos % P.q_cap);
    if (seq != pos + 1) return ~0ull;
    // an item published for another search of the team (that rank is ahead or behind): skip
    const uint32_t ep = ((const volatile uint32_t *)P.team_items[r])[(pos % P.q_cap) * kItemWords + 5];
    if (ep != P.epoch) return ~0ull;
    return atomicCAS_system(&RC->q_head, pos, pos + 1) == pos ? pos : ~0ull;
}

// 1-D bulk copy (TMA engine) global -> shared, completing on an mbarrier with a tx count
__device__ __forceinline__ void mbar_init(unsigned long long *mbar) {
    const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_stage(uint32_t *dst, const uint32_t *src, uint32_t bytes, unsigned long long *mbar) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst), m = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");      // generic reads of the last use first
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src), "r"(bytes), "r"(m) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *mbar, uint32_t parity) {
    const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(m), "r"(parity) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One level l of a warp's DFS stack (§4.2, Alg. 2 S[l][lane]).  448 bytes; 416 with the
// slice length and source level packed in one word (GM_PACK_CS: lengths < 2^27, a degree
// bound gm_count checks; source levels < 31, and 31 marks a sibling-buffer slice); 384 when
// also the parent lane rides in the top 5 bits of the vertex word (PK: the 16/24/32-level
// kernels with GM_PACK_PID, vertex ids < 2^27, checked by gm_count).
template <bool PK>
struct StackPid { uint8_t pid[32]; };   // S[l][lane].pid : parent lane at level l-1
template <>
struct StackPid<true> {};
template <bool PK>
struct alignas(16) StackLevel : StackPid<PK> {
    uint32_t v[32];       // S[l][lane].v   : candidate data vertex of the task in this lane (PK: | pid << 27)
    uint32_t cb[32];      // S[l][lane].C   : begin of the local candidate slice of lane's partial match
#if GM_PACK_CS
    uint32_t clcs[32];    //                  its length | (source level << 27)
#else
    uint32_t cl[32];      //                  its length
    uint8_t cs[32];       //                  level whose vertex produced the slice (its check is implied)
#endif
    static constexpr uint32_t kLow27 = (1u << 27) - 1;
    __device__ __forceinline__ uint32_t vtx(uint32_t j) const {
        if constexpr (PK) return v[j] & kLow27; else return v[j];
    }
    __device__ __forceinline__ uint32_t par(uint32_t j) const {
        if constexpr (PK) return v[j] >> 27; else return this->pid[j];
    }
    __device__ __forceinline__ void set_vp(uint32_t j, uint32_t x, uint32_t p) {
        if constexpr (PK) v[j] = x | (p << 27); else { v[j] = x; this->pid[j] = (uint8_t)p; }
    }
#if GM_PACK_CS
    __device__ __forceinline__ uint32_t len(uint32_t j) const { return clcs[j] & kLow27; }
    __device__ __forceinline__ uint32_t src(uint32_t j) const { return clcs[j] >> 27; }
    __device__ __forceinline__ void set(uint32_t j, uint32_t n, uint32_t s) { clcs[j] = n | (s << 27); }
    __device__ __forceinline__ void set_len(uint32_t j, uint32_t n) { clcs[j] = (clcs[j] & ~kLow27) | n; }
#else
    __device__ __forceinline__ uint32_t len(uint32_t j) const { return cl[j]; }
    __device__ __forceinline__ uint32_t src(uint32_t j) const { return cs[j]; }
    __device__ __forceinline__ void set(uint32_t j, uint32_t n, uint32_t s) { cl[j] = n; cs[j] = (uint8_t)s; }
    __device__ __forceinline__ void set_len(uint32_t j, uint32_t n) { cl[j] = n; }
#endif
};

// A warp's shared-memory state: a fixed header, then the stack levels.  Only the levels a
// query's search touches are allocated (SearchParams.levels, host-computed: the counted
// last one or two levels of set / pair counting hold nothing), and the per-warp scratch rows
// -- check images and set/pair-counting words, sized per query (SearchParams.rows_chk /
// rows_last) -- follow them: so a query of fewer than D vertices, or one that counts its
// last levels, keeps more warps resident on the shared-memory-limited 16/24/32-level kernels.
template <int D>
struct alignas(16) WarpStack {
    unsigned long long mbar;  // GM_TWO_STAGE: mbarrier of the warp's bulk-copy staging buffer
    uint32_t home;            // gm_team: lineage rank of the unit this warp holds
    uint32_t sibn[D <= 8 ? 32 : 1];   // sibling prefixes (8-level kernels only): siblings per parent lane
    uint32_t ci[D];       // virtual-task-pool cursor: source lane ...
    uint32_t cj[D];       // ... and offset inside its slice (§4.2 "two lightweight pointers")
    using Level = StackLevel<(D > 8 && GM_PACK_PID != 0)>;
    Level lv[D];          // levels 0 .. SearchParams.levels - 1 are allocated
};

// GenerateTask (Alg. 2 lines 17-24, Erratum 2 read as a running minimum): the local
// candidate set of the partial match ending at (l-1, lane) is the label-L(phi[l]) slice
// of N(M[u']) for the backward neighbour u' with the fewest such neighbours (§4.1).
template <int D>
__device__ __forceinline__ void generate(const SearchParams &P, WarpStack<D> &S, int l, bool valid, uint32_t lane,
                                         uint32_t &words) {
    uint32_t best = 0, cb = 0, cs = 0;
    if (valid) {
        const uint32_t bw = P.bw[l];
        const uint32_t lab = P.lab[l];
        const uint32_t gt = P.sb_gt[l], lt = P.sb_lt[l];
        const int lowest = __ffs(bw | gt | lt) - 1;
        best = 0xffffffffu;
        uint32_t lb = 0, ub = 0xffffffffu;     // symmetry breaking: candidates in [lb, ub)
        uint32_t p = lane;
        if (GM_CUT_MIN && (gt | lt)) {
            // The bounds cut every backward row to [lb, ub); the fewest candidates are in the
            // row whose CUT is shortest, which on degree-ordered ids is often not the shortest
            // row (a low-degree vertex's neighbours are mostly high-degree, i.e. small ids).
            // First the bounds, then each row's cut by two binary searches.
            for (int i = l - 1; i >= lowest; --i) {
                const uint32_t w = S.lv[i].vtx(p);
                if ((gt >> i) & 1u) lb = max(lb, w + 1);
                if ((lt >> i) & 1u) ub = min(ub, w);
                p = S.lv[i].par(p);
            }
            p = lane;
            for (int i = l - 1; i >= lowest; --i) {
                if ((bw >> i) & 1u) {
                    const uint32_t row = S.lv[i].vtx(p) * P.S + lab;
                    const uint32_t lo = ld_nc(P.offs + row), len = ld_nc(P.offs + row + 1) - lo;
                    words += 2;
                    if (lb < ub && len) {
                        const uint32_t a = lb ? lower_bound_idx(P.nbr + lo, len, lb, words) : 0u;
                        const uint32_t e = ub != 0xffffffffu ? a + lower_bound_idx(P.nbr + lo + a, len - a, ub, words) : len;
                        if (e - a < best) { best = e - a; cb = lo + a; cs = (uint32_t)i; }
                    } else {
                        best = 0; cb = lo; cs = (uint32_t)i;
                    }
                }
                p = S.lv[i].par(p);
            }
        } else {
            for (int i = l - 1; i >= lowest; --i) {
                const uint32_t w = S.lv[i].vtx(p);
                if ((bw >> i) & 1u) {
                    const uint32_t row = w * P.S + lab;
                    const uint32_t lo = ld_nc(P.offs + row), hi = ld_nc(P.offs + row + 1);
                    words += 2;
                    if (hi - lo < best) { best = hi - lo; cb = lo; cs = (uint32_t)i; }
                }
                if ((gt >> i) & 1u) lb = max(lb, w + 1);
                if ((lt >> i) & 1u) ub = min(ub, w);
                p = S.lv[i].par(p);
            }
            if (gt | lt) {   // the slice is sorted: cut it to the ids the conditions allow
                uint32_t a = 0, e = best;
                if (lb > 0 && best) a = lower_bound_idx(P.nbr + cb, best, lb, words);
                if (ub != 0xffffffffu && best) e = lower_bound_idx(P.nbr + cb, best, ub, words);
                cb += a;
                best = e > a ? e - a : 0;
            }
        }
    }
    S.lv[l].cb[lane] = cb;
    S.lv[l].set(lane, best, cs);
}

// GenerateTask with a per-grandparent part (GM_GEN_CACHE).  At level l = P.gen_level (the
// level holding most tasks) every passing task of level l-1 calls GenerateTask, but the rows
// of its backward neighbours mapped at levels <= l-2, and the symmetry bounds from those
// levels, are the same for all children of one level-(l-2) partial match.  gen_prep computes
// that part once per level-(l-2) lane when level l-1 is entered: the shortest such row, cut to
// those bounds (GENW rows 0-2: begin, length, source level; rows 3-4: the bounds).  Then
// generate_cached only looks at the row of level l-1 (when phi[l-1] is a backward neighbour)
// and level l-1's bounds: the cached cut slice, cut further by them, or the level-(l-1) row
// if its full length is shorter, cut by all bounds.  Any backward neighbour's row cut to the
// bounds is a superset of the feasible set (§4.1), so either choice is exact.
template <int D>
__device__ __forceinline__ void gen_prep(const SearchParams &P, WarpStack<D> &S, uint32_t *__restrict__ scr, bool valid,
                                         uint32_t lane, uint32_t &words) {
    if (!valid) return;
    const int l = (int)P.gen_level;
    const uint32_t below = (1u << (l - 1)) - 1;            // levels <= l-2
    const uint32_t bw = P.bw[l] & below, gt = P.sb_gt[l] & below, lt = P.sb_lt[l] & below;
    const uint32_t lab = P.lab[l];
    uint32_t best = 0xffffffffu, cb = 0, cs = 0, lb = 0, ub = 0xffffffffu;
    const int lowest = __ffs(bw | gt | lt) - 1;
    uint32_t p = lane;
    for (int i = l - 2; i >= lowest && lowest >= 0; --i) {
        const uint32_t w = S.lv[i].vtx(p);
        if ((bw >> i) & 1u) {
            const uint32_t row = w * P.S + lab;
            const uint32_t lo = ld_nc(P.offs + row), hi = ld_nc(P.offs + row + 1);
            words += 2;
            if (hi - lo < best) { best = hi - lo; cb = lo; cs = (uint32_t)i; }
        }
        if ((gt >> i) & 1u) lb = max(lb, w + 1);
        if ((lt >> i) & 1u) ub = min(ub, w);
        p = S.lv[i].par(p);
    }
    if (bw && (gt | lt)) {
        uint32_t a = 0, e = best;
        if (lb > 0 && best) a = lower_bound_idx(P.nbr + cb, best, lb, words);
        if (ub != 0xffffffffu && best) e = lower_bound_idx(P.nbr + cb, best, ub, words);
        cb += a;
        best = e > a ? e - a : 0;
    }
    GENW(0, lane) = cb; GENW(1, lane) = best; GENW(2, lane) = cs; GENW(3, lane) = lb; GENW(4, lane) = ub;
}

template <int D>
__device__ __forceinline__ void generate_cached(const SearchParams &P, WarpStack<D> &S, uint32_t *__restrict__ scr, int l,
                                                bool valid, uint32_t lane, uint32_t &words) {
    uint32_t best = 0, cb = 0, cs = 0;
    if (valid) {
        const uint32_t p = S.lv[l - 1].par(lane);
        const uint32_t v1 = S.lv[l - 1].vtx(lane);
        const uint32_t nb = (P.bw[l] >> (l - 1)) & 1u;
        const uint32_t ngt = (P.sb_gt[l] >> (l - 1)) & 1u, nlt = (P.sb_lt[l] >> (l - 1)) & 1u;
        cb = GENW(0, p); best = GENW(1, p); cs = GENW(2, p);
        uint32_t lo = 0, len = 0xffffffffu;
        if (nb) {
            const uint32_t row = v1 * P.S + P.lab[l];
            lo = ld_nc(P.offs + row); len = ld_nc(P.offs + row + 1) - lo;
            words += 2;
        }
        if (len < best) {
            // the level-(l-1) row is shorter than the cached cut: cut it to every bound
            const uint32_t lb = max(GENW(3, p), ngt ? v1 + 1 : 0u), ub = min(GENW(4, p), nlt ? v1 : 0xffffffffu);
            uint32_t a = 0, e = len;
            if (lb >= ub) { e = 0; }
            else {
                if (lb > 0 && len) a = lower_bound_idx(P.nbr + lo, len, lb, words);
                if (ub != 0xffffffffu && len) e = lower_bound_idx(P.nbr + lo, len, ub, words);
            }
            cb = lo + a; best = e > a ? e - a : 0; cs = (uint32_t)(l - 1);
        } else if (ngt | nlt) {
            // the cached slice (already cut to the far bounds), cut to level l-1's bound
            uint32_t a = 0, e = best;
            if (ngt && best) a = lower_bound_idx(P.nbr + cb, best, v1 + 1, words);
            if (nlt && best) e = lower_bound_idx(P.nbr + cb, best, v1, words);
            cb += a;
            best = e > a ? e - a : 0;
        }
    }
    S.lv[l].cb[lane] = cb;
    S.lv[l].set(lane, best, cs);
}

// Process (Alg. 2 lines 32-41, Erratum 1 read as "lanes without a task return false"):
// candidate-filter bit, then one walk up the pid chain checking injectivity and, for each
// backward neighbour other than the slice's source, adjacency by binary search.
//
// Called by all 32 lanes together (lanes without a task pass has = false) and written to
// stay converged: the pid-chain walk has the same trip count in every lane, the checks
// run in a uniform loop over the (uniform) number of backward neighbours, and the binary
// searches step in lock-step until every lane is done (instead of per-lane early exits
// that leave most of the warp idle; ncu measured 12 active lanes/warp before).
template <int D, bool SIB>
__device__ __forceinline__ bool process(const SearchParams &P, WarpStack<D> &S, uint32_t *__restrict__ scr, int l, uint32_t v, uint32_t src,
                                        bool has, uint32_t lane, bool par, uint32_t &words) {
    // The candidate-bitmap word is loaded first and tested after the chain walk, so its L2
    // round trip overlaps the walk; it still gates the (costlier) adjacency probes.
    uint32_t cword = 0xffffffffu;
    if (has && ((P.cand_needed >> l) & 1u)) {
        cword = ld_nc(P.cand + P.candoff[l] + (v >> 5));
        ++words;
    }
    bool ok = has;
    const uint32_t cs = has ? S.lv[l].src(src) : 0u;
    const uint32_t chk = has ? P.bw[l] & ~(1u << cs) : 0u;   // exactly nchk images for a task
    const uint32_t lab = P.lab[l];
    // Only levels holding a backward neighbour (adjacency check) or a vertex of v's label
    // (v can only collide with a same-label image) need visiting; the walk stops at the
    // deepest such level, uniformly across lanes (P.walk_low[l]).
    const uint32_t eq = P.same_lab[l], gt = P.sb_gt[l], lt = P.sb_lt[l];
    const int nchk = __popc(P.bw[l]) - 1;           // uniform (the source level is in bw)
    // par: the set-counting level, whose checks prep_last stored per parent lane (CHK(., src)).
    // There, injectivity only needs the same-label images that are not backward neighbours
    // (v in N(w) implies v != w), and the symmetry-breaking bounds were applied to the slice
    // by generate().  Elsewhere one walk up the pid chain collects the checks per task.
    const uint32_t ccol = par ? src : lane;
    if (par) {
        const int neq = __popc(eq & ~P.bw[l]);
        for (int e = 0; e < neq; ++e) ok = ok && (CHK(nchk + e, src) != v);
    } else {
        uint32_t p = src;
        int k = 0;
        // (ordering hub checks first measured 1-7 % slower on rmat18 dense queries: pairs of
        // mixed hub/search probes overlap better)
        for (int i = l - 1; i >= (int)P.walk_low[l]; --i) {   // injectivity + collect the checks
            const uint32_t w = S.lv[i].vtx(p);
            if ((eq >> i) & 1u) ok = ok && (w != v);
            if ((gt >> i) & 1u) ok = ok && (v > w);            // symmetry-breaking conditions
            if ((lt >> i) & 1u) ok = ok && (v < w);
            if ((chk >> i) & 1u) { CHK(k, lane) = w; ++k; }
            p = S.lv[i].par(p);
        }
    }
    ok = ok && ((cword >> (v & 31)) & 1u);          // filter verdict gates the probes below
    // G checks per pass: their hub-id, bitmap/row-offset and binary-search loads are
    // independent, so each lane keeps G dependent-load chains in flight (the L2-resident
    // 8-level kernel is bound by long-scoreboard stalls on its probes: G = 2).  A larger G
    // wastes the probes of tasks that fail an earlier check of the group (most do), which on
    // the DRAM-resident configs costs more than the overlap gains: G = 1 for 16/32 levels.
    constexpr int G = D <= 8 ? 2 : GM_PROBES_WIDE;
    for (int c = 0; c < nchk; c += G) {
        if (!__any_sync(FULL, ok)) break;
        uint32_t w[G], b[G], n[G], hh[G], hx[G], sw[G];
        bool r[G], need[G], hub[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            w[g] = (ok && c + g < nchk) ? CHK(c + g, ccol) : 0u;
            const bool act = ok && c + g < nchk && !(SIB && w[g] == ~0u);   // (~0u: no check, sibling prefix)
            r[g] = true; need[g] = false; hub[g] = false; b[g] = 0; n[g] = 0; hh[g] = 0; hx[g] = 0;
            sw[g] = 0xffffffffu;
            if (act) {
                // hub bitmap of w, or of v (the test is symmetric), else binary search of w's row
                if (w[g] < P.nhubs || (GM_VHUB && v < P.nhubs)) {
                    hh[g] = w[g] < P.nhubs ? w[g] : v;
                    hx[g] = w[g] < P.nhubs ? v : w[g];
                    hub[g] = true;
                    sw[g] = hub_summ_word<(D > 8)>(P, hh[g], hx[g], words);   // (summary level: first load)
                } else {
                    const uint32_t row = w[g] * P.S + lab;
                    b[g] = ld_nc(P.offs + row);
                    n[g] = ld_nc(P.offs + row + 1) - b[g];
                    need[g] = true;
                    words += 2;
                }
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {       // bitmap words, only where the summary bit is set
            if (hub[g]) {
                if (summ_says(sw[g], hx[g])) {
                    ++words;
                    r[g] = (ld_nc(P.hub_bits + (unsigned long long)hh[g] * P.hub_words + (hx[g] >> 5)) >> (hx[g] & 31)) & 1u;
                } else {
                    r[g] = false;
                }
            }
        }
        bool more = false;
#pragma unroll
        for (int g = 0; g < G; ++g) more = more || n[g] > 1;
        while (__any_sync(FULL, more)) {   // lock-step branch-free lower bounds
            more = false;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                if (n[g] > 1) {
                    const uint32_t half = n[g] >> 1;
                    b[g] = (ld_nc(P.nbr + b[g] + half) <= v) ? b[g] + half : b[g];
                    n[g] -= half;
                    ++words;
                    more = more || n[g] > 1;
                }
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if (need[g]) { r[g] = n[g] == 1 && ld_nc(P.nbr + b[g]) == v; words += n[g]; }
            ok = ok && r[g];
        }
    }
    return ok;
}

// Process for T tasks per lane at a terminal per-parent level (wide rounds, GM_WIDE): the
// same checks as process(..., par = true) -- filter bit, same-label injectivity against the
// parent's list, one adjacency check per pass -- for tasks (v[t], src[t]) in lock step, so
// every lane keeps T independent probe chains in flight, all of them needed (unlike a second
// check of one task, which is wasted when the first fails).
template <int D, int T, bool SIB>
__device__ __forceinline__ void process_parT(const SearchParams &P, WarpStack<D> &S, uint32_t *__restrict__ scr, int l,
                                             const uint32_t (&v)[T], const uint32_t (&src)[T], const bool (&has)[T],
                                             bool (&F)[T], uint32_t &words) {
    uint32_t cw[T];
    const bool filt = (P.cand_needed >> l) & 1u;
#pragma unroll
    for (int t = 0; t < T; ++t) {
        cw[t] = 0xffffffffu;
        if (filt && has[t]) { cw[t] = ld_nc(P.cand + P.candoff[l] + (v[t] >> 5)); ++words; }
    }
    bool ok[T];
#pragma unroll
    for (int t = 0; t < T; ++t) ok[t] = has[t];
    const uint32_t lab = P.lab[l];
    const int nchk = __popc(P.bw[l]) - 1;
    const int neq = __popc(P.same_lab[l] & ~P.bw[l]);
    for (int e = 0; e < neq; ++e) {
#pragma unroll
        for (int t = 0; t < T; ++t) ok[t] = ok[t] && (CHK(nchk + e, src[t]) != v[t]);
    }
    bool any = false;
#pragma unroll
    for (int t = 0; t < T; ++t) {
        ok[t] = ok[t] && ((cw[t] >> (v[t] & 31)) & 1u);
        any = any || ok[t];
    }
    for (int c = 0; c < nchk; ++c) {
        if (!__any_sync(FULL, any)) break;
        uint32_t b[T], n[T], sw[T], hh[T], hx[T];
        bool r[T], need[T], hub[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            b[t] = 0; n[t] = 0; sw[t] = 0xffffffffu; hh[t] = 0; hx[t] = 0;
            r[t] = true; need[t] = false; hub[t] = false;
            if (!ok[t]) continue;
            const uint32_t w = CHK(c, src[t]);
            if (SIB && w == ~0u) continue;           // no check in this row (sibling prefix)
            if (w < P.nhubs || (GM_VHUB && v[t] < P.nhubs)) {
                hh[t] = w < P.nhubs ? w : v[t];
                hx[t] = w < P.nhubs ? v[t] : w;
                hub[t] = true;
                sw[t] = hub_summ_word<(D > 8)>(P, hh[t], hx[t], words);
            } else {
                const uint32_t row = w * P.S + lab;
                b[t] = ld_nc(P.offs + row);
                n[t] = ld_nc(P.offs + row + 1) - b[t];
                need[t] = true;
                words += 2;
            }
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
            if (hub[t]) {
                if (summ_says(sw[t], hx[t])) {
                    ++words;
                    r[t] = (ld_nc(P.hub_bits + (unsigned long long)hh[t] * P.hub_words + (hx[t] >> 5)) >> (hx[t] & 31)) & 1u;
                } else {
                    r[t] = false;
                }
            }
        }
        bool more = false;
#pragma unroll
        for (int t = 0; t < T; ++t) more = more || n[t] > 1;
        while (__any_sync(FULL, more)) {
            more = false;
#pragma unroll
            for (int t = 0; t < T; ++t) {
                if (n[t] > 1) {
                    const uint32_t half = n[t] >> 1;
                    b[t] = (ld_nc(P.nbr + b[t] + half) <= v[t]) ? b[t] + half : b[t];
                    n[t] -= half;
                    ++words;
                    more = more || n[t] > 1;
                }
            }
        }
        any = false;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            if (need[t]) { r[t] = n[t] == 1 && ld_nc(P.nbr + b[t]) == v[t]; words += n[t]; }
            ok[t] = ok[t] && r[t];
            any = any || ok[t];
        }
    }
#pragma unroll
    for (int t = 0; t < T; ++t) F[t] = ok[t];
}

// The checks of the tasks at level l = P.par_level (the level holding almost all tasks: the
// set-counting level, else the last), recorded once per parent lane when the level is
// entered, so that process() reads them by src instead of walking the pid chain per task:
// the backward images other than the slice's source, then the same-label images that are
// not backward neighbours (the only ones injectivity must compare: v in N(w) implies v != w).
template <int D, bool SIB>
__device__ __forceinline__ void prep_checks(const SearchParams &P, WarpStack<D> &S, uint32_t *__restrict__ scr, int l, bool valid,
                                            uint32_t lane) {
    if (!valid) return;
    // a sibling-prefix slice (sib_append) already satisfies every check of phi[l-1] -- adjacency
    // to its backward images, injectivity against the same-label images below, its bounds --
    // so only the positions in sib_chk remain; unused rows hold ~0u ("no check": no vertex has
    // that id, process() skips it and injectivity never matches it)
    const bool sibl = SIB && (uint32_t)l == P.sib_level && S.lv[l].src(lane) == kSibCs;
    const uint32_t chkm = sibl ? P.sib_chk : P.bw[l] & ~(1u << S.lv[l].src(lane));
    const uint32_t eqm = sibl ? 0u : P.same_lab[l] & ~P.bw[l];
    const int nchk = __popc(P.bw[l]) - 1;
    int kc = 0, ke = 0;
    uint32_t p = lane;
    for (int i = l - 1; i >= (int)P.par_low; --i) {
        const uint32_t w = S.lv[i].vtx(p);
        if ((chkm >> i) & 1u) { CHK(kc, lane) = w; ++kc; }
        if ((eqm >> i) & 1u) { CHK(nchk + ke, lane) = w; ++ke; }
        p = S.lv[i].par(p);
    }
    if (SIB && P.sib_level) {
        for (int k = kc; k < nchk; ++k) CHK(k, lane) = ~0u;
        const int neq = __popc(P.same_lab[l] & ~P.bw[l]);
        for (int e = ke; e < neq; ++e) CHK(nchk + e, lane) = ~0u;
    }
#if GM_CHK_ORDER
    // most selective check first: larger device id = lower degree = fewer neighbours, so more
    // tasks fail early and whole warps leave the probe loop sooner
    // (GM_CHK_HUBFIRST, 16/32-level kernels: hubs first -- on DRAM-resident graphs a failing
    // hub test costs one bitmap sector, a failing search the row offsets plus the search)
    auto key = [&](uint32_t x) { return (GM_CHK_HUBFIRST && D > 8 && x < P.nhubs) ? (x | 0x80000000u) : x; };
    for (int a = 1; a < kc; ++a) {
        const uint32_t x = CHK(a, lane), kx = key(x);
        int b = a - 1;
        while (b >= 0 && key(CHK(b, lane)) < kx) { CHK(b + 1, lane) = CHK(b, lane); --b; }
        CHK(b + 1, lane) = x;
    }
#endif
}

// Sibling prefixes (count mode).  When phi[s] (s = P.sib_level, the last
// position) is adjacent to phi[s-1] and to every backward neighbour of phi[s-1], has its label,
// a candidate filter no stricter, and symmetry-breaking bounds that include M[phi[s]] <
// M[phi[s-1]] and every bound of phi[s-1], then every valid image of phi[s] is a valid image
// of phi[s-1] under the same parent M[0..s-2] that is smaller than M[phi[s-1]].  Those
// siblings were all validated before M[phi[s-1]] itself (a slice is dealt in ascending
// order), so recording each parent's valid siblings in order gives, for the task v that
// just passed at level s-1, a complete candidate slice: the recorded prefix before v.  Its
// tasks need only the checks in P.sib_chk (adjacency to v and to the backward neighbours
// phi[s-1] lacks), against the |N(M[u'])|-long slice of §4.1 with every check.
// Called by all lanes at the descent from level s-1 (v, src: the task of this lane at level
// s-1 and its parent lane; F: it passed): records v and returns its position in the parent's
// list, i.e. the length of its prefix (a lane at position >= sib_cap keeps generate's slice:
// the buffer holds only the first sib_cap siblings).
template <int D>
__device__ __forceinline__ uint32_t sib_append(const SearchParams &P, WarpStack<D> &S, uint32_t v, uint32_t src,
                                               bool F, uint32_t lane, uint32_t sib_base) {
    const uint32_t grp = __match_any_sync(FULL, F ? src : 32u + lane);   // passing lanes per parent
    const uint32_t pos = (F ? S.sibn[src] : 0u) + __popc(grp & ((1u << lane) - 1));
    __syncwarp();
    if (F) {
        if (pos < P.sib_cap) P.sib[sib_base + src * P.sib_cap + pos] = v;
        if ((grp >> lane) == 1u) S.sibn[src] = pos + 1;   // the group's highest lane
    }
    __syncwarp();
    return pos;
}

// Candidate `off` of the slice of (level l, parent lane src): the CSR, or (sibling prefixes)
// the warp's sibling buffer -- written during this launch, so read with a coherent load
template <int D, bool SIB>
__device__ __forceinline__ uint32_t cand_at(const SearchParams &P, const WarpStack<D> &S, int l, uint32_t src, uint32_t off) {
    const uint32_t cb = S.lv[l].cb[src];
    if (SIB && P.sib_level == (uint32_t)l && S.lv[l].src(src) == kSibCs) return P.sib[cb + off];
    return ld_nc(P.nbr + cb + off);
}

// Last-level set counting (count mode): when phi[last] has ONE
// backward neighbour phi[b], the valid extensions of a partial match M of depth last are
// exactly the vertices of N_{L(phi[last])}(M[b]) not already in M (adjacency is the only
// edge constraint; the candidate filter is implied -- every such v completes an embedding,
// so it passes any sound filter).  A mapped M[i] can lie in that slice only if
// L(phi[i]) = L(phi[last]) (bitmask same_lab); it surely does if phi[i] ~ phi[b] in Q
// (adj_b), else one binary search decides.  Cost O(|M|) instead of O(|slice|) tasks.
// (l, v, src) is the task that just completed M at level l = last - 1.
//
// The part that depends only on the parent (levels < l) is computed once per parent lane when
// level l = last-1 is entered (prep_last), not once per task: M[b] when b < l, and the
// same-label images not adjacent to phi[b] in Q (those need an adjacency test).
template <int D>
__device__ __forceinline__ void prep_last(const SearchParams &P, WarpStack<D> &S, uint32_t *__restrict__ scr, int l, bool valid, uint32_t lane,
                                          uint32_t &words) {
    if (!valid) return;
    const int b = (int)P.last_b;
    const uint32_t test = P.last_same & ~P.last_adj;
    const uint32_t known = P.last_sb ? (P.last_same & P.last_adj) : 0u;   // parked only with bounds
    const uint32_t gt = P.sb_gt[l + 1], lt = P.sb_lt[l + 1];
    uint32_t mb = 0, lb = 0, ub = 0xffffffffu;
    int k = 0, ka = 0;
    uint32_t p = lane;
    for (int i = l - 1; i >= (int)P.last_low; --i) {
        const uint32_t w = S.lv[i].vtx(p);
        if (i == b) mb = w;
        if ((test >> i) & 1u) { LASTW(k, lane) = w; ++k; }
        if ((known >> i) & 1u) { LASTW(P.last_k + ka, lane) = w; ++ka; }
        if ((gt >> i) & 1u) lb = max(lb, w + 1);
        if ((lt >> i) & 1u) ub = min(ub, w);
        p = S.lv[i].par(p);
    }
    AUXW(0, lane) = mb;
    AUXW(1, lane) = lb;
    AUXW(2, lane) = ub;
    if (b < l && !P.last_sb) {
        // M[b] is fixed for this parent: the count of every task is this constant minus (at
        // most) the task's own vertex; keep it in lastlb (bounds are unused without SB)
        const uint32_t lab = P.lab[l + 1];
        const uint32_t row = mb * P.S + lab;
        uint32_t cnt = ld_nc(P.offs + row + 1) - ld_nc(P.offs + row) -
                       (uint32_t)__popc(P.last_same & P.last_adj & ((2u << l) - 1));
        words += 2;
        for (int c = 0; c < k; ++c)
            if (has_edge<(D > 8)>(P, mb, P.lab[b], LASTW(c, lane), lab, words)) --cnt;
        AUXW(1, lane) = cnt;
    }
}

template <int D>
__device__ __forceinline__ uint32_t count_last(const SearchParams &P, const WarpStack<D> &S, uint32_t *__restrict__ scr, int l, uint32_t v,
                                               uint32_t src, uint32_t &words) {
    const uint32_t lab = P.lab[l + 1];
    const uint32_t same = P.last_same;    // positions i < last, i != b, with L(phi[i]) == lab
    const uint32_t mb = (int)P.last_b == l ? v : AUXW(0, src);   // M[b]
    const uint32_t lb_lab = P.lab[P.last_b];                       // L(M[b])
    if (!P.last_sb && (int)P.last_b < l) {   // parent-constant part precomputed by prep_last
        uint32_t cnt = AUXW(1, src);
        if (((same >> l) & 1u) && !((P.last_adj >> l) & 1u) && has_edge<(D > 8)>(P, mb, lb_lab, v, lab, words)) --cnt;
        return cnt;
    }
    const uint32_t row = mb * P.S + lab;
    const uint32_t lo = ld_nc(P.offs + row), hi = ld_nc(P.offs + row + 1);
    words += 2;
    if (P.last_sb) {
        // symmetry breaking bounds phi[last]'s image to [lb, ub): count that part of the sorted
        // slice, then remove the mapped same-label vertices inside it
        uint32_t lb = AUXW(1, src), ub = AUXW(2, src);
        if ((P.sb_gt[l + 1] >> l) & 1u) lb = max(lb, v + 1);
        if ((P.sb_lt[l + 1] >> l) & 1u) ub = min(ub, v);
        if (lb >= ub) return 0;
        const uint32_t len = hi - lo;
        const uint32_t a = lb ? lower_bound_idx(P.nbr + lo, len, lb, words) : 0u;
        const uint32_t e = ub != 0xffffffffu ? lower_bound_idx(P.nbr + lo, len, ub, words) : len;
        uint32_t cnt = e > a ? e - a : 0u;
        if (((same >> l) & 1u) && v >= lb && v < ub &&
            (((P.last_adj >> l) & 1u) || has_edge<(D > 8)>(P, mb, lb_lab, v, lab, words)))
            --cnt;
        for (uint32_t c = 0; c < P.last_k; ++c) {
            const uint32_t w = LASTW(c, src);
            if (w >= lb && w < ub && has_edge<(D > 8)>(P, mb, lb_lab, w, lab, words)) --cnt;
        }
        for (uint32_t c = 0; c < P.last_ka; ++c) {
            const uint32_t w = LASTW(P.last_k + c, src);
            if (w >= lb && w < ub) --cnt;
        }
        return cnt;
    }
    // mapped vertices adjacent to phi[b] in Q lie in the slice for sure (same label)
    uint32_t cnt = hi - lo - (uint32_t)__popc(same & P.last_adj & ((2u << l) - 1));
    if (((same >> l) & 1u) && !((P.last_adj >> l) & 1u) && has_edge<(D > 8)>(P, mb, lb_lab, v, lab, words)) --cnt;
    for (uint32_t c = 0; c < P.last_k; ++c)
        if (has_edge<(D > 8)>(P, mb, lb_lab, LASTW(c, src), lab, words)) --cnt;
    return cnt;
}

// Per-parent part of pair counting, run when level l = last-2 is entered: M[b6], M[b7] and
// the bounds of A = N(M[b6]) and R = N(M[b7]) when those are parent images (b < l), and the
// mapped same-label images (levels < l) inside A, inside R and inside both.  The images'
// membership is only summed here when no per-task row needs them (!P.two_walk).
template <int D>
__device__ __forceinline__ void prep_two(const SearchParams &P, WarpStack<D> &S, uint32_t *__restrict__ scr, int l, bool valid, uint32_t lane,
                                         uint32_t &words) {
    if (!valid) return;
    const uint32_t lab6 = P.lab[l + 1], lab7 = P.lab[l + 2];
    const int b6 = (int)P.two_b6, b7 = (int)P.two_b7;
    uint32_t m6 = 0, m7 = 0;
    uint32_t p = lane;
    for (int i = l - 1; i >= (int)P.two_low; --i) {
        const uint32_t w = S.lv[i].vtx(p);
        if (i == b6) m6 = w;
        if (i == b7) m7 = w;
        p = S.lv[i].par(p);
    }
    LASTW(0, lane) = m6;
    LASTW(1, lane) = m7;
    if (b6 < l) {
        const uint32_t ra = m6 * P.S + lab6;
        LASTW(2, lane) = ld_nc(P.offs + ra); LASTW(3, lane) = ld_nc(P.offs + ra + 1);
        words += 2;
    }
    if (b7 < l) {
        const uint32_t rr = m7 * P.S + lab7;
        LASTW(4, lane) = ld_nc(P.offs + rr); LASTW(5, lane) = ld_nc(P.offs + rr + 1);
        words += 2;
    }
    uint32_t inA = 0, inR = 0, inAR = 0;
    if (!P.two_walk) {
        p = lane;
        for (int i = l - 1; i >= (int)P.two_low; --i) {
            const uint32_t w = S.lv[i].vtx(p);
            bool a = false, r = false;
            if ((P.two_same6 >> i) & 1u) a = ((P.two_adj6 >> i) & 1u) || has_edge<(D > 8)>(P, m6, P.lab[b6], w, lab6, words);
            if ((P.two_same7 >> i) & 1u) r = ((P.two_adj7 >> i) & 1u) || has_edge<(D > 8)>(P, m7, P.lab[b7], w, lab7, words);
            inA += a; inR += r; inAR += a && r;
            p = S.lv[i].par(p);
        }
    }
    AUXW(0, lane) = inA;
    AUXW(1, lane) = inR;
    AUXW(2, lane) = inAR;
}

// Pair counting (count mode): when phi[last-1] and phi[last] each
// have ONE backward neighbour, b6 and b7, and are not adjacent to each other, the embeddings
// extending a partial match M of depth last-1 (levels 0..l, l = last-2) are the pairs
// (x, y) with x in A = N_{L(phi[last-1])}(M[b6]), y in R = N_{L(phi[last])}(M[b7]), neither
// mapped in M, and x != y.  (Adjacency to the single backward neighbour is the only edge
// constraint on each; both candidate filters are implied, as for count_last.)  With
// V = A \ M and B = |R \ M|:
//     count = |V| * B - [L(phi[last-1]) == L(phi[last])] * |V n R|,
//     |V n R| = |A n R| - |M n A n R|,
// where |A n R| (b6 != b7) is one sorted-list intersection, computed by the whole warp
// (shorter list split over the lanes, each element tested against the longer list's hub
// bitmap or by binary search).  Warp-collective: every lane calls it; F = lane has a valid
// partial match ending in (l, v, src).  ISECT = false compiles the intersection out (callers
// that only run it for leaves of different labels: the wide rounds).
template <int D, bool ISECT = true>
__device__ __forceinline__ unsigned long long count_two(const SearchParams &P, WarpStack<D> &S, uint32_t *__restrict__ scr, int l,
                                                        uint32_t v, uint32_t src, bool F, uint32_t lane,
                                                        uint32_t &words, uint32_t &stage_phase) {
    const uint32_t lab6 = P.lab[l + 1], lab7 = P.lab[l + 2];
    const int b6 = (int)P.two_b6, b7 = (int)P.two_b7;
    uint32_t m6 = v, m7 = v, a0 = 0, a1 = 0, r0 = 0, r1 = 0, inA = 0, inR = 0, inAR = 0;
    if (F) {
        // parent-constant parts from prep_two (lastw rows 0-5, lastmb/lb/ub); the row of a
        // backward neighbour mapped at this level (b == l, i.e. v) is read per task
        if (b6 < l) { m6 = LASTW(0, src); a0 = LASTW(2, src); a1 = LASTW(3, src); }
        else { const uint32_t ra = v * P.S + lab6; a0 = ld_nc(P.offs + ra); a1 = ld_nc(P.offs + ra + 1); words += 2; }
        if (b7 < l) { m7 = LASTW(1, src); r0 = LASTW(4, src); r1 = LASTW(5, src); }
        else { const uint32_t rr = v * P.S + lab7; r0 = ld_nc(P.offs + rr); r1 = ld_nc(P.offs + rr + 1); words += 2; }
        // mapped vertices inside A and R: only same-label ones can be; surely if their query
        // vertex is adjacent to phi[b] in Q, else one edge test
        if (P.two_walk) {       // a per-task row with same-label images below l: test them all here
            uint32_t p = src;
            for (int i = l - 1; i >= (int)P.two_low; --i) {
                const uint32_t w = S.lv[i].vtx(p);
                bool a = false, r = false;
                if ((P.two_same6 >> i) & 1u) a = ((P.two_adj6 >> i) & 1u) || has_edge<(D > 8)>(P, m6, P.lab[b6], w, lab6, words);
                if ((P.two_same7 >> i) & 1u) r = ((P.two_adj7 >> i) & 1u) || has_edge<(D > 8)>(P, m7, P.lab[b7], w, lab7, words);
                inA += a; inR += r; inAR += a && r;
                p = S.lv[i].par(p);
            }
        } else {                // every image below l was tested once per parent
            inA = AUXW(0, src); inR = AUXW(1, src); inAR = AUXW(2, src);
        }
        {   // the task's own vertex (never in a row it owns: same6/same7 exclude b6/b7)
            bool a = false, r = false;
            if ((P.two_same6 >> l) & 1u) a = ((P.two_adj6 >> l) & 1u) || has_edge<(D > 8)>(P, m6, P.lab[b6], v, lab6, words);
            if ((P.two_same7 >> l) & 1u) r = ((P.two_adj7 >> l) & 1u) || has_edge<(D > 8)>(P, m7, P.lab[b7], v, lab7, words);
            inA += a; inR += r; inAR += a && r;
        }
    }
    const unsigned long long nV = (unsigned long long)(a1 - a0 - inA), nB = (unsigned long long)(r1 - r0 - inR);
    unsigned long long cnt = nV * nB;
    if (ISECT && lab6 == lab7) {              // uniform
        unsigned long long ar = 0;
        if (b6 == b7) {
            ar = a1 - a0;                     // A == R
        } else {
            // segmented intersection: the shorter lists of all lanes form one virtual pool of
            // elements, dealt 32 per round like ScatterTask; each element is tested against its
            // owner's longer list (hub bitmap, else binary search); hits are summed per owner
            const bool a_short = a1 - a0 <= r1 - r0;
            const uint32_t sb = a_short ? a0 : r0, sl = F ? (a_short ? a1 - a0 : r1 - r0) : 0u;
            const uint32_t gb = a_short ? r0 : a0, ge = a_short ? r1 : a1, gown = a_short ? m7 : m6;
            AUXW(3, lane) = 0;
            __syncwarp();
            uint32_t ci = 0, cj = 0;
#if GM_TWO_STAGE
            uint32_t *stage = &LASTW(P.two_stage_row, 0);   // kStageWords words after the pair-count rows
            uint32_t stage_tag = ~0u;                       // aligned start of the staged list
#endif
            while (true) {
                // fast path: the cursor's list alone fills the round (long lists against a hub)
                const uint32_t sl_ci = __shfl_sync(FULL, sl, ci & 31);
#if GM_TWO_VEC8 && !GM_TWO_STAGE
                if (ci < 32 && sl_ci - cj >= 256) {
                    // 256 elements per round: two 16-byte loads per lane and 8 independent
                    // probes in flight (the 128-element round below, twice as wide)
                    const uint32_t f_sb = __shfl_sync(FULL, sb, ci), f_gb = __shfl_sync(FULL, gb, ci);
                    const uint32_t f_ge = __shfl_sync(FULL, ge, ci), f_gown = __shfl_sync(FULL, gown, ci);
                    const uint32_t start = f_sb + cj, a = start & ~3u;
                    const uint4 q0 = __ldg(reinterpret_cast<const uint4 *>(P.nbr + a) + lane);
                    const uint4 q1 = __ldg(reinterpret_cast<const uint4 *>(P.nbr + a + 128) + lane);
                    const uint32_t x[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
                    bool hit[8];
                    uint32_t nval = 0;
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        hit[g] = a + 128 * (g >> 2) + 4 * lane + (g & 3) >= start;
                        nval += hit[g];
                    }
                    words += nval;
                    if (f_gown < P.nhubs) {
                        const uint32_t *row = P.hub_bits + (unsigned long long)f_gown * P.hub_words;
                        uint32_t wv[8];
#pragma unroll
                        for (int g = 0; g < 8; ++g) wv[g] = hit[g] ? hub_summ_word<(D > 8)>(P, f_gown, x[g], words) : 0u;
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            hit[g] = hit[g] && summ_says(wv[g], x[g]);
                            if (hit[g]) { wv[g] = ld_nc(row + (x[g] >> 5)); ++words; }
                        }
#pragma unroll
                        for (int g = 0; g < 8; ++g) hit[g] = hit[g] && ((wv[g] >> (x[g] & 31)) & 1u);
                    } else {
                        uint32_t n = f_ge - f_gb, b[8];
#pragma unroll
                        for (int g = 0; g < 8; ++g) b[g] = f_gb;
                        while (n > 1) {
                            const uint32_t half = n >> 1;
#pragma unroll
                            for (int g = 0; g < 8; ++g) b[g] = (ld_nc(P.nbr + b[g] + half) <= x[g]) ? b[g] + half : b[g];
                            n -= half;
                            words += nval;
                        }
#pragma unroll
                        for (int g = 0; g < 8; ++g) hit[g] = hit[g] && n == 1 && ld_nc(P.nbr + b[g]) == x[g];
                        words += nval;
                    }
                    uint32_t h = 0;
#pragma unroll
                    for (int g = 0; g < 8; ++g) h += __popc(__ballot_sync(FULL, hit[g]));
                    if (lane == 0) AUXW(3, ci) += h;
                    __syncwarp();
                    cj += a + 256 - start;
                    if (cj == sl_ci) { ++ci; cj = 0; }
                    continue;
                }
#endif
#if GM_TWO_VEC
                if (ci < 32 && sl_ci - cj >= 128) {
                    // 128 elements per round with one 16-byte load per lane (LDG.E.128): lane j
                    // takes the 4 words at a + 4j of the aligned block [a, a + 128) that holds
                    // the cursor (words before the cursor are masked; a + 128 <= the list's end
                    // because >= 128 remain), and keeps 4 independent probes in flight.  The
                    // elements form a set, so the order they are tested in is immaterial.
                    const uint32_t f_sb = __shfl_sync(FULL, sb, ci), f_gb = __shfl_sync(FULL, gb, ci);
                    const uint32_t f_ge = __shfl_sync(FULL, ge, ci), f_gown = __shfl_sync(FULL, gown, ci);
                    const uint32_t start = f_sb + cj, a = start & ~3u;
                    const uint4 q4 = __ldg(reinterpret_cast<const uint4 *>(P.nbr + a) + lane);
                    const uint32_t x[4] = {q4.x, q4.y, q4.z, q4.w};
                    bool hit[4];
                    uint32_t nval = 0;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        hit[g] = a + 4 * lane + g >= start;
                        nval += hit[g];
                    }
                    words += nval;
                    if (f_gown < P.nhubs) {
                        const uint32_t *row = P.hub_bits + (unsigned long long)f_gown * P.hub_words;
                        uint32_t wv[4];
#pragma unroll
                        for (int g = 0; g < 4; ++g) wv[g] = hit[g] ? hub_summ_word<(D > 8)>(P, f_gown, x[g], words) : 0u;
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            hit[g] = hit[g] && summ_says(wv[g], x[g]);
                            if (hit[g]) { wv[g] = ld_nc(row + (x[g] >> 5)); ++words; }
                        }
#pragma unroll
                        for (int g = 0; g < 4; ++g) hit[g] = hit[g] && ((wv[g] >> (x[g] & 31)) & 1u);
                    } else {
                        // four lower bounds in the same list: the trip count is warp-uniform
                        uint32_t n = f_ge - f_gb, b[4] = {f_gb, f_gb, f_gb, f_gb};
#if GM_TWO_STAGE
                        const uint32_t *L = P.nbr;
                        if (n && n <= kStageWords - 6) {   // the aligned superset fits the buffer
                            const uint32_t a0 = f_gb & ~3u;
                            if (a0 != stage_tag) {
                                __syncwarp();
                                if (lane == 0)
                                    bulk_stage(stage, P.nbr + a0, 4u * (((f_ge + 3u) & ~3u) - a0), &S.mbar);
                                mbar_wait(&S.mbar, stage_phase);
                                stage_phase ^= 1u;
                                stage_tag = a0;
                            }
                            L = stage - a0;                  // L[i] = nbr[i] for i in [a0, end)
                        }
#define GM_LD_L(i) (L[i])
#else
#define GM_LD_L(i) ld_nc(P.nbr + (i))
#endif
                        while (n > 1) {
                            const uint32_t half = n >> 1;
#pragma unroll
                            for (int g = 0; g < 4; ++g) b[g] = (GM_LD_L(b[g] + half) <= x[g]) ? b[g] + half : b[g];
                            n -= half;
                            words += nval;
                        }
#pragma unroll
                        for (int g = 0; g < 4; ++g) hit[g] = hit[g] && n == 1 && GM_LD_L(b[g]) == x[g];
                        words += nval;
#undef GM_LD_L
                    }
                    uint32_t h = 0;
#pragma unroll
                    for (int g = 0; g < 4; ++g) h += __popc(__ballot_sync(FULL, hit[g]));
                    if (lane == 0) AUXW(3, ci) += h;
                    __syncwarp();
                    cj += a + 128 - start;
                    if (cj == sl_ci) { ++ci; cj = 0; }
                    continue;
                }
#endif
                if (ci < 32 && sl_ci - cj >= 32) {
                    const uint32_t f_sb = __shfl_sync(FULL, sb, ci), f_gb = __shfl_sync(FULL, gb, ci);
                    const uint32_t f_ge = __shfl_sync(FULL, ge, ci), f_gown = __shfl_sync(FULL, gown, ci);
                    // two elements per lane when 64 remain: two independent probes in flight
                    const uint32_t step = sl_ci - cj >= 64 ? 64u : 32u;
                    const uint32_t x = ld_nc(P.nbr + f_sb + cj + lane);
                    const uint32_t x2 = step == 64 ? ld_nc(P.nbr + f_sb + cj + 32 + lane) : 0u;
                    words += step >> 5;
                    bool hit, hit2 = false;
                    if (f_gown < P.nhubs) {
                        const uint32_t *row = P.hub_bits + (unsigned long long)f_gown * P.hub_words;
                        const uint32_t s1 = hub_summ_word<(D > 8)>(P, f_gown, x, words);
                        const uint32_t s2 = step == 64 ? hub_summ_word<(D > 8)>(P, f_gown, x2, words) : 0u;
                        const bool p1 = summ_says(s1, x), p2 = step == 64 && summ_says(s2, x2);
                        const uint32_t w1 = p1 ? ld_nc(row + (x >> 5)) : 0u;
                        const uint32_t w2 = p2 ? ld_nc(row + (x2 >> 5)) : 0u;
                        words += p1 + p2;
                        hit = (w1 >> (x & 31)) & 1u;
                        hit2 = (w2 >> (x2 & 31)) & 1u;
                    } else {
                        hit = contains(P.nbr, f_gb, f_ge, x, words);
                        if (step == 64) hit2 = contains(P.nbr, f_gb, f_ge, x2, words);
                    }
                    const uint32_t h = __popc(__ballot_sync(FULL, hit)) + __popc(__ballot_sync(FULL, hit2));
                    if (lane == 0) AUXW(3, ci) += h;
                    __syncwarp();
                    cj += step;
                    if (cj == sl_ci) { ++ci; cj = 0; }
                    continue;
                }
                uint32_t rem = lane >= ci ? sl - (lane == ci ? cj : 0u) : 0u;
                const uint32_t r32 = min(rem, 32u);
                uint32_t incl = r32;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t x = __shfl_up_sync(FULL, incl, o);
                    if (lane >= (uint32_t)o) incl += x;
                }
                const uint32_t total = __shfl_sync(FULL, incl, 31);
                if (total == 0) break;
                const uint32_t k = min(total, 32u);
                uint32_t src = 0;
#pragma unroll
                for (uint32_t bb = 16; bb >= 1; bb >>= 1) {
                    const uint32_t x = __shfl_sync(FULL, incl, src + bb - 1);
                    if (x <= lane) src += bb;
                }
                src = min(src, 31u);
                const uint32_t src_excl = __shfl_sync(FULL, incl - r32, src);
                const uint32_t off = lane < k ? lane - src_excl + (src == ci ? cj : 0u) : 0u;
                const uint32_t s_sb = __shfl_sync(FULL, sb, src), s_gb = __shfl_sync(FULL, gb, src);
                const uint32_t s_ge = __shfl_sync(FULL, ge, src), s_gown = __shfl_sync(FULL, gown, src);
                const uint32_t lsrc = __shfl_sync(FULL, src, k - 1), loff = __shfl_sync(FULL, off, k - 1);
                const uint32_t lsl = __shfl_sync(FULL, sl, lsrc);
                if (loff + 1 < lsl) { ci = lsrc; cj = loff + 1; } else { ci = lsrc + 1; cj = 0; }
                if (lane < k) {
                    const uint32_t x = ld_nc(P.nbr + s_sb + off);
                    ++words;
                    bool hit;
                    if (s_gown < P.nhubs) {
                        hit = hub_bit<(D > 8)>(P, s_gown, x, words);
                    } else {
                        hit = contains(P.nbr, s_gb, s_ge, x, words);
                    }
                    if (hit) atomicAdd(&AUXW(3, src), 1u);
                }
            }
            __syncwarp();
            ar = AUXW(3, lane);
        }
        if (F) cnt -= ar - inAR;
    }
    return F ? cnt : 0ull;
}

// Walk the chain of (level, lane) and write the prefix M[0..level] into dst (by position).
template <int D>
__device__ __forceinline__ void read_prefix(const WarpStack<D> &S, int level, uint32_t lane, uint32_t *dst) {
    uint32_t p = lane;
    for (int i = level; i >= 0; --i) {
        dst[i] = S.lv[i].vtx(p);
        p = S.lv[i].par(p);
    }
}

// ------------------------------------------------------------------ DFS kernel

// WORDS: count the algorithmic words read (gm_run_stats.words, GM_FLAG_COUNT_WORDS).  The
// counters are per-probe register adds in the hot loops; with WORDS = false they are dead code
// and the compiler removes them (measured 12-23 % more throughput), so the timed
// searches run without them and the bench takes words per task from a separate counting pass.
// SIB: the code for symmetric unlabelled-style patterns is compiled in -- sibling prefixes
// (sib_append) and the cached GenerateTask part (gen_prep); the instantiations without it keep
// their register budget and code size (the 8-level kernel spilled with it, and the other
// queries lost 10-30 % to the larger code).
// MODE: which counting code is compiled in -- kModePlain (none: every level by tasks),
// kModeSet (last-level set counting), kModePair (set + pair counting), kModePat (the pattern
// code: sibling prefixes, cached GenerateTask part; 8 levels, no set counting).  Each query
// runs the smallest kernel holding its paths: a kernel's size is mostly code a given query
// never runs, and the instruction-cache misses it causes cost 14-18 % on the rmat18 dense
// queries (the pair-counting split).
template <int D, bool ENUM, bool WORDS, int MODE>
__global__ void __launch_bounds__(dfs_max_warps<D>() * 32, GM_DFS_MINB_D(D)) k_dfs(const SearchParams P) {
    constexpr bool SIB = MODE == kModePat;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t *wbase = smem_raw + (size_t)(threadIdx.x >> 5) * P.warp_stride;
    WarpStack<D> &S = *reinterpret_cast<WarpStack<D> *>(wbase);
    uint32_t *__restrict__ scr = reinterpret_cast<uint32_t *>(wbase + P.stack_bytes);
    const uint32_t lane = threadIdx.x & 31;
    const int last = (int)P.nq - 1;
    // this warp's sibling buffer (32 parent lanes x sib_cap words)
    const uint32_t sibL = SIB ? P.sib_level : 0u;
    const uint32_t bulk_two = MODE == kModePair ? P.bulk_two : 0u;    // (compiled in per MODE)
    const uint32_t bulk_last = (MODE == kModeSet || MODE == kModePair) ? P.bulk_last : 0u;
    const uint32_t sib_base = SIB ? (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32u * P.sib_cap : 0u;
    Ctrl *C = P.ctrl;
    volatile Ctrl *VC = C;

    unsigned long long my_count = 0, my_tasks = 0, my_rounds = 0, my_don = 0, my_words = 0;
    bool ovf = false;          // my_count wrapped (add_count)
    uint32_t stage_phase = 0;  // GM_TWO_STAGE: parity of the staging mbarrier's next phase
#if GM_TWO_STAGE
    if (P.two_stage_row && lane == 0) mbar_init(&S.mbar);
    __syncwarp();
#endif
    uint32_t wacc = 0;
    uint32_t tick = 0;
    bool stop = false;
    // (the lineage rank of the unit this warp holds, gm_team, lives in S.home: read only on a
    // donation and at the unit's end, it need not occupy a register through the search)
    // time limit relative to this launch: the first warp to start stamps t0
    if (P.limit_ns && lane == 0) atomicCAS(&C->t0, 0ull, globaltimer());

    while (!stop) {
        // ------------------------------------------------ acquire a unit of work
        int base = 0, l = 0;
        bool got = false;
        uint32_t backoff = 64;
        uint32_t src_rank = P.team_rank;     // ring the popped item came from
        bool registered = false;             // this idle warp has posted a steal request
        uint32_t idle_polls = 0;             // failed polls since then (team: remote requests)
        while (true) {
            unsigned long long b = ~0ull, item = ~0ull;
            int exit_now = 0;
            if (lane == 0) {
                if (VC->abort) {
                    exit_now = 1;
                } else if (!P.no_pool && pool_peek(P) < P.pool_size) {
                    work_add(P, C, P.team_rank, 1);
                    // P.pool_ctr: this launch's counter, or one shared by every rank's launch
                    // (peer memory over NVLink: multi-GPU dynamic chunk assignment)
                    b = pool_claim(P, (unsigned long long)P.batch);
                    if (b >= P.pool_size) { work_add(P, C, P.team_rank, -1); b = ~0ull; }
                }
                if (!exit_now && b == ~0ull) {
                    if (!P.steal) {
                        exit_now = 1;
                    } else {
                        if (!registered) { req_add(P, C, 1); registered = true; idle_polls = 0; }
                        // pop (bounded MPMC ring, per-slot sequence numbers): own ring first,
                        // then (team) the other ranks' rings over peer memory
                        item = ring_pop(P, C, P.team_rank);
                        src_rank = P.team_rank;
                        for (uint32_t k = 1; k < GM_TEAMN(P) && item == ~0ull; ++k) {
                            src_rank = (P.team_rank + k) % GM_TEAMN(P);
                            item = ring_pop(P, C, src_rank);
                        }
                        if (item == ~0ull && GM_TEAMN(P) > 1 && (++idle_polls & 31u) == 0) {
                            // still idle: ask the next rank's busy warps to split their stacks
                            const uint32_t r = (P.team_rank + 1 + (idle_polls >> 5) % (GM_TEAMN(P) - 1)) % GM_TEAMN(P);
                            atomicAdd_system(&P.team_ctrl[r]->requests, 1);
                        }
                        if (item == ~0ull && pool_peek(P) >= P.pool_size && team_idle(P, VC))
                            exit_now = 1;
                    }
                }
                if (b != ~0ull || item != ~0ull) registered = false;
            }
            b = __shfl_sync(FULL, b, 0);
            item = __shfl_sync(FULL, item, 0);
            src_rank = __shfl_sync(FULL, src_rank, 0);
            exit_now = __shfl_sync(FULL, exit_now, 0);
            if (exit_now) { stop = true; break; }
            if (b != ~0ull) {
                if (lane == 0) S.home = P.team_rank;   // a pool batch: this rank's lineage
                // pool batch: up to `batch` partial matches of depth d0 become the lanes of level d0-1
                const unsigned long long k = min((unsigned long long)P.batch, P.pool_size - b);
                const bool valid = lane < k;
                const int d0 = (int)P.d0;
                for (int i = 0; i < d0; ++i) {
                    S.lv[i].set_vp(lane, valid ? P.pool[(unsigned long long)i * P.pool_size + b + lane] : 0u, lane);
                }
                __syncwarp();
                generate<D>(P, S, d0, valid, lane, wacc);
                if (d0 + 1 == (int)sibL) S.sibn[lane] = 0;
                if (GM_GEN_CACHE && SIB && d0 + 1 == (int)P.gen_level) gen_prep<D>(P, S, scr, valid, lane, wacc);
                if (d0 == (int)P.par_level) prep_checks<D, SIB>(P, S, scr, d0, valid, lane);
                if (!ENUM && bulk_two && d0 == last - 2) prep_two<D>(P, S, scr, d0, valid, lane, wacc);
                if (!ENUM && bulk_last && d0 == last - 1) prep_last<D>(P, S, scr, d0, valid, lane, wacc);
                base = d0; l = d0;
                got = true;
                break;
            }
            if (item != ~0ull) {
                // lane 0's acquire load of the slot's sequence number, then this warp barrier
                // (memory-ordering among the lanes), then every lane's strong item loads
                if (GM_TEAMN(P)) __threadfence_system(); else __threadfence();
                __syncwarp();
                const unsigned long long slot = item % P.q_cap;
                // written by another SM (or, in a team, another GPU): volatile loads, which
                // are strong at system scope (LDG.E.STRONG.SYS), never a stale L1 line
                const volatile uint32_t *it =
                    (GM_TEAMN(P) ? P.team_items[src_rank] : P.q_items) + slot * kItemWords;
                const uint32_t depth = it[0];
                if (lane < depth) S.lv[lane].set_vp(0, it[6 + lane], 0);
                S.lv[depth].cb[lane] = lane == 0 ? it[1] : 0;
                S.lv[depth].set(lane, lane == 0 ? it[2] : 0u, lane == 0 ? it[3] : 0u);
                if (lane == 0) S.home = it[4];
                __syncwarp();
                if (lane == 0) {   // release the slot for the next lap of the ring
                    if (GM_TEAMN(P)) {
                        __threadfence_system();
                        ((volatile unsigned long long *)P.team_seq[src_rank])[slot] = item + P.q_cap;
                    } else {
                        __threadfence();
                        ((volatile unsigned long long *)P.q_seq)[slot] = item + P.q_cap;
                    }
                }
                if ((int)depth + 1 == (int)sibL) S.sibn[lane] = 0;
                if (GM_GEN_CACHE && SIB && (int)depth + 1 == (int)P.gen_level) gen_prep<D>(P, S, scr, lane == 0, lane, wacc);
                if ((int)depth == (int)P.par_level) prep_checks<D, SIB>(P, S, scr, depth, lane == 0, lane);
                if (!ENUM && bulk_two && (int)depth == last - 2) prep_two<D>(P, S, scr, depth, lane == 0, lane, wacc);
                if (!ENUM && bulk_last && (int)depth == last - 1) prep_last<D>(P, S, scr, depth, lane == 0, lane, wacc);
                base = (int)depth; l = (int)depth;
                got = true;
                break;
            }
            __nanosleep(backoff);
            backoff = min(backoff * 2, 8192u);
        }
        if (!got) break;
        if (lane == 0) { S.ci[l] = 0; S.cj[l] = 0; }
        __syncwarp();

        // ------------------------------------------------ depth-first batch exploration
        while (l >= base) {
            if (((++tick) & 31u) == 0) {
                int ab = 0, claim = 0;
                if (lane == 0) {
                    if (P.limit_ns && globaltimer() > VC->t0 + P.limit_ns) atomicExch(&C->abort, 1);
                    ab = VC->abort;
                    // work stealing (§4.3): serve one posted request by splitting our stack
                    if (P.steal && (GM_TEAMN(P) ? ld_sys(&C->requests) : VC->requests) > 0) {
                        if (req_add(P, C, -1) > 0) claim = 1;
                        else req_add(P, C, 1);
                    }
                }
                if (__shfl_sync(FULL, ab, 0)) { stop = true; break; }
                if (__shfl_sync(FULL, claim, 0)) {
                    // shallowest level with splittable untouched work (the last level's tasks
                    // are single checks: never worth a hand-off)
                    int served = 0;
                    // (sibling prefixes: neither level sib-1, whose siblings a parent records in
                    // order, nor level sib, whose slices live in this warp's buffer)
                    const int top = min(l, sibL ? (int)sibL - 2 : last - 1);
                    for (int s = base; s <= top && !served; ++s) {
                        const uint32_t ci = S.ci[s], cj = S.cj[s];
                        if (ci >= 32) continue;
                        const uint32_t cl = S.lv[s].len(lane);
                        // worth a hand-off: >= 2 levels left below s, or >= 256 untouched tasks
                        const uint32_t myrem = lane > ci ? cl : (lane == ci ? cl - cj : 0u);
                        const uint32_t remtot = __reduce_add_sync(FULL, min(myrem, 1u << 20));
                        if (last - s < 2 && remtot < 256) continue;
                        const uint32_t mask = __ballot_sync(FULL, lane > ci && cl > 0);
                        uint32_t giver = 32, keep = 0, give = 0, gb = 0;
                        if (mask) {                       // hand off the last untouched parent lane
                            giver = 31 - __clz(mask);
                            give = __shfl_sync(FULL, cl, giver);
                        } else {
                            const uint32_t rem = S.lv[s].len(ci) - cj;
                            if (rem >= 2) { giver = ci; keep = rem / 2; give = rem - keep; gb = cj + keep; }
                        }
                        if (giver == 32) continue;
                        // reserve a ring slot
                        unsigned long long pos = ~0ull;
                        if (lane == 0) {
                            work_add(P, C, S.home, 1);        // the new unit keeps this unit's lineage
                            pos = VC->q_tail;
                            while (true) {
                                // (slots are released by poppers, possibly on other GPUs)
                                const unsigned long long seq = GM_TEAMN(P) ? ld_acq_sys(P.q_seq + pos % P.q_cap)
                                                                        : ((volatile unsigned long long *)P.q_seq)[pos % P.q_cap];
                                if (seq == pos) {
                                    const unsigned long long prev = atomicCAS(&C->q_tail, pos, pos + 1);
                                    if (prev == pos) break;
                                    pos = prev;
                                } else if (seq < pos) {       // full
                                    pos = ~0ull;
                                    break;
                                } else {
                                    pos = VC->q_tail;
                                }
                            }
                            if (pos == ~0ull) work_add(P, C, S.home, -1);
                        }
                        pos = __shfl_sync(FULL, pos, 0);
                        if (pos == ~0ull) break;          // ring full: keep the work
                        if (lane == giver) {
                            uint32_t *it = P.q_items + (pos % P.q_cap) * kItemWords;
                            it[0] = (uint32_t)s; it[1] = S.lv[s].cb[giver] + gb; it[2] = give; it[3] = S.lv[s].src(giver);
                            it[4] = S.home; it[5] = P.epoch;
                            read_prefix<D>(S, s - 1, giver, it + 6);
                            S.lv[s].set_len(giver, mask ? 0u : gb);
                            if (GM_TEAMN(P)) __threadfence_system(); else __threadfence();
                            ((volatile unsigned long long *)P.q_seq)[pos % P.q_cap] = pos + 1;
                        }
                        served = 1;
                        my_don += (lane == 0);
                    }
                    if (!served && lane == 0) req_add(P, C, 1);   // give the request back
                    __syncwarp();
                }
            }

#if GM_WIDE
            // ---- wide round: at the terminal per-parent level (the set-counting level, else the
            // last level; nothing descends from it) each lane takes WT tasks of the virtual task
            // pool, lane + 32 j (ScatterTask over 32 WT slots), and validates them in lock step
            // (process_parT): WT independent probe chains per lane, no probe wasted, and the
            // per-round overheads (scatter, control checks, counting) paid once per 32 WT tasks.
            // (also the pair-counting level when the two leaves have different labels: count_two
            // is then per task, without the warp-collective intersection)
            if (D >= GM_WIDE_MIN_D && !ENUM && l == (int)P.par_level &&
                (bulk_two ? (GM_WIDE_PAIR && l == last - 2 && P.lab[last - 1] != P.lab[last])
                            : (l == last || (bulk_last && l == last - 1)))) {
                constexpr int WT = D > 16 ? GM_WIDE_T32 : (D > 8 ? GM_WIDE_T16 : (SIB ? GM_WIDE_TSIB : GM_WIDE_T));
                const uint32_t ci = S.ci[l], cj = S.cj[l];
                uint32_t tsrc[WT], toff[WT], k;
                const uint32_t cl_ci = ci < 32 ? S.lv[l].len(ci) : 0u;
                if (ci < 32 && cl_ci - cj >= 32u * WT) {
#pragma unroll
                    for (int t = 0; t < WT; ++t) { tsrc[t] = ci; toff[t] = cj + 32u * t + lane; }
                    k = 32u * WT;
                    if (lane == 0) {
                        if (cj + 32u * WT < cl_ci) S.cj[l] = cj + 32u * WT;
                        else { S.ci[l] = ci + 1; S.cj[l] = 0; }
                    }
                } else {
                    uint32_t rem = 0;
                    if (lane >= ci) rem = S.lv[l].len(lane) - (lane == ci ? cj : 0);
                    const uint32_t rw = min(rem, 32u * WT);
                    uint32_t incl = rw;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t x = __shfl_up_sync(FULL, incl, o);
                        if (lane >= (uint32_t)o) incl += x;
                    }
                    const uint32_t total = __shfl_sync(FULL, incl, 31);
                    if (total == 0) { --l; continue; }       // level exhausted: backtrack
                    k = min(total, 32u * WT);
                    // source lane of task t = number of lanes whose inclusive count is <= t
#pragma unroll
                    for (int t = 0; t < WT; ++t) tsrc[t] = 0;
#pragma unroll
                    for (uint32_t bb = 16; bb >= 1; bb >>= 1) {
#pragma unroll
                        for (int t = 0; t < WT; ++t)
                            if (__shfl_sync(FULL, incl, tsrc[t] + bb - 1) <= lane + 32u * t) tsrc[t] += bb;
                    }
#pragma unroll
                    for (int t = 0; t < WT; ++t) {
                        tsrc[t] = min(tsrc[t], 31u);
                        const uint32_t ex = __shfl_sync(FULL, incl - rw, tsrc[t]);
                        const uint32_t tt = lane + 32u * t;
                        toff[t] = tt < k ? tt - ex + (tsrc[t] == ci ? cj : 0) : 0;
                    }
                    // cursor after task k-1 (held by lane (k-1) % 32 in slot (k-1) / 32)
                    const uint32_t lt = (k - 1) & 31u, lj = (k - 1) >> 5;
                    uint32_t ls = tsrc[0], lo = toff[0];
#pragma unroll
                    for (int t = 1; t < WT; ++t)
                        if (lj == (uint32_t)t) { ls = tsrc[t]; lo = toff[t]; }
                    const uint32_t lsrc = __shfl_sync(FULL, ls, lt), loff = __shfl_sync(FULL, lo, lt);
                    if (lane == 0) {
                        if (loff + 1 < S.lv[l].len(lsrc)) { S.ci[l] = lsrc; S.cj[l] = loff + 1; }
                        else { S.ci[l] = lsrc + 1; S.cj[l] = 0; }
                    }
                }
                uint32_t tv[WT];
                bool th[WT], tf[WT];
                uint32_t nh = 0;
#pragma unroll
                for (int t = 0; t < WT; ++t) {
                    th[t] = lane + 32u * t < k;
                    tv[t] = th[t] ? cand_at<D, SIB>(P, S, l, tsrc[t], toff[t]) : 0;
                    nh += th[t];
                }
                my_rounds += (lane == 0) ? (uint32_t)WT : 0u;   // 32 WT task slots (idle rate)
                my_tasks += nh;
#if GM_PREFETCH_ROWS
                // the counting step after the checks reads the task vertex's own row offsets (pair
                // counting with a leaf on this level, set counting with phi[last]'s backward
                // neighbour on it): start those loads now so they overlap the checks
                if (bulk_two || bulk_last) {
                    const uint32_t pl = bulk_two ? ((int)P.two_b6 == l ? P.lab[l + 1] : ((int)P.two_b7 == l ? P.lab[l + 2] : ~0u))
                                                 : ((int)P.last_b == l ? P.lab[l + 1] : ~0u);
                    if (pl != ~0u) {
#pragma unroll
                        for (int t = 0; t < WT; ++t)
                            if (th[t]) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.offs + tv[t] * P.S + pl));
                    }
                }
#endif
                process_parT<D, WT, SIB>(P, S, scr, l, tv, tsrc, th, tf, wacc);
#ifdef GM_LEVEL_STATS
                {
                    uint32_t np = 0;
#pragma unroll
                    for (int t = 0; t < WT; ++t) np += __popc(__ballot_sync(FULL, tf[t]));
                    if (lane == 0) { atomicAdd(&g_level_tasks[l], (unsigned long long)k); atomicAdd(&g_level_pass[l], (unsigned long long)np); }
                }
#endif
                GM_ADD_WORDS(wacc + nh);
                wacc = 0;
                if (l == last) {
#pragma unroll
                    for (int t = 0; t < WT; ++t) my_count += tf[t];
                } else if (GM_WIDE_LOOP_D(D)) {
                    // one copy of count_two / count_last in a loop body instead of WT unrolled
                    // copies (code size is an instruction-cache cost: ncu no_instruction stalls)
#pragma unroll 1
                    for (int t = 0; t < WT; ++t) {
                        uint32_t vt = tv[0], st = tsrc[0];
                        bool ft = tf[0];
#pragma unroll
                        for (int u = 1; u < WT; ++u)
                            if (t == u) { vt = tv[u]; st = tsrc[u]; ft = tf[u]; }
                        if (bulk_two)
                            add_count(my_count, count_two<D, false>(P, S, scr, l, vt, st, ft, lane, wacc, stage_phase), ovf);
                        else if (ft)
                            add_count(my_count, count_last<D>(P, S, scr, l, vt, st, wacc), ovf);
                    }
                } else if (bulk_two) {
                    // (different-label leaves only: count_two without its intersection)
#pragma unroll
                    for (int t = 0; t < WT; ++t)
                        add_count(my_count, count_two<D, false>(P, S, scr, l, tv[t], tsrc[t], tf[t], lane, wacc, stage_phase), ovf);
                } else {
#pragma unroll
                    for (int t = 0; t < WT; ++t)
                        if (tf[t]) add_count(my_count, count_last<D>(P, S, scr, l, tv[t], tsrc[t], wacc), ovf);
                }
                __syncwarp();
                continue;
            }
#endif
            // ---- ScatterTask, warp-parallel: next 32 tasks of the virtual task pool at level l
            const uint32_t ci = S.ci[l], cj = S.cj[l];
            uint32_t src, off, k;
            const uint32_t cl_ci = ci < 32 ? S.lv[l].len(ci) : 0u;
            if (cl_ci - cj >= 32 && ci < 32) {
                // fast path: the cursor's slice alone fills the batch (long slices, hubs)
                src = ci; off = cj + lane; k = 32;
                if (lane == 0) {
                    if (cj + 32 < cl_ci) S.cj[l] = cj + 32;
                    else { S.ci[l] = ci + 1; S.cj[l] = 0; }
                }
            } else {
                uint32_t rem = 0;
                if (lane >= ci) rem = S.lv[l].len(lane) - (lane == ci ? cj : 0);
                const uint32_t r32 = min(rem, 32u);
                uint32_t incl = r32;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t x = __shfl_up_sync(FULL, incl, o);
                    if (lane >= (uint32_t)o) incl += x;
                }
                const uint32_t total = __shfl_sync(FULL, incl, 31);
                if (total == 0) { --l; continue; }       // level exhausted: backtrack
                k = min(total, 32u);
                // source lane of task `lane` = number of lanes whose inclusive count is <= lane
                src = 0;
#pragma unroll
                for (uint32_t b = 16; b >= 1; b >>= 1) {
                    const uint32_t x = __shfl_sync(FULL, incl, src + b - 1);
                    if (x <= lane) src += b;
                }
                src = min(src, 31u);
                const uint32_t src_excl = __shfl_sync(FULL, incl - r32, src);
                off = lane < k ? lane - src_excl + (src == ci ? cj : 0) : 0;
                const uint32_t lsrc = __shfl_sync(FULL, src, k - 1);
                const uint32_t loff = __shfl_sync(FULL, off, k - 1);
                if (lane == 0) {
                    if (loff + 1 < S.lv[l].len(lsrc)) { S.ci[l] = lsrc; S.cj[l] = loff + 1; }
                    else { S.ci[l] = lsrc + 1; S.cj[l] = 0; }
                }
            }
            const bool has = lane < k;
            const uint32_t v = has ? cand_at<D, SIB>(P, S, l, src, off) : 0;
            my_rounds += (lane == 0);
            my_tasks += has;
#ifdef GM_LEVEL_STATS
            if (lane == 0) atomicAdd(&g_level_tasks[l], (unsigned long long)k);
#endif

            // ---- Process
            const bool F = process<D, SIB>(P, S, scr, l, v, src, has, lane, l == (int)P.par_level, wacc);
#ifdef GM_LEVEL_STATS
            if (lane == 0) atomicAdd(&g_level_pass[l], (unsigned long long)__popc(__ballot_sync(FULL, F)));
            else __ballot_sync(FULL, F);
#endif
            GM_ADD_WORDS(wacc + (has ? 1u : 0u));
            wacc = 0;
            if (!ENUM && bulk_two && l == last - 2) {
                // pair counting: both remaining levels of every partial match at once
                add_count(my_count, count_two<D>(P, S, scr, l, v, src, F, lane, wacc, stage_phase), ovf);
                __syncwarp();
                continue;
            }
            if (l == last) {
                if (ENUM) {
                    const uint32_t fm = __ballot_sync(FULL, F);
                    unsigned long long basepos = 0;
                    if (lane == 0 && fm) {
                        basepos = atomicAdd(&C->out_ctr, (unsigned long long)__popc(fm));
                        // GM_FLAG_STOP_AT_CAPACITY: the buffer is full, stop the search
                        if (P.stop_at_cap && basepos + __popc(fm) >= P.out_cap) atomicExch(&C->abort, 1);
                    }
                    basepos = __shfl_sync(FULL, basepos, 0);
                    if (F) {
                        const unsigned long long idx = basepos + __popc(fm & ((1u << lane) - 1));
                        if (idx < P.out_cap) {
                            uint32_t *row = P.out + idx * P.nq;
                            row[P.col[l]] = ld_nc(P.new2old + v);        // original ids out
                            uint32_t p = src;
                            for (int i = l - 1; i >= 0; --i) {
                                row[P.col[i]] = ld_nc(P.new2old + S.lv[i].vtx(p));
                                p = S.lv[i].par(p);
                            }
                        }
                    }
                }
                my_count += F;
                __syncwarp();
                continue;
            }
            if (!ENUM && bulk_last && l == last - 1) {
                // last-level set counting: the extensions of this partial match are exactly the
                // label-L(phi[last]) neighbours of its backward neighbour minus the mapped ones
                if (F) add_count(my_count, count_last<D>(P, S, scr, l, v, src, wacc), ovf);
                __syncwarp();
                continue;
            }
            if (has) S.lv[l].set_vp(lane, v, src);
            const uint32_t fm = __ballot_sync(FULL, F);
            __syncwarp();
            if (!fm) continue;
            // ---- descend: GenerateTask for level l+1 on the lanes that extended
            if (SIB && l + 1 == (int)sibL) {
                // sibling prefix when the buffer holds it (no GenerateTask), else the usual slice
                const uint32_t pos = sib_append<D>(P, S, v, src, F, lane, sib_base);
                const bool sibok = F && pos < P.sib_cap;
                generate<D>(P, S, l + 1, F && !sibok, lane, wacc);
                if (sibok) {
                    S.lv[l + 1].cb[lane] = sib_base + src * P.sib_cap; S.lv[l + 1].set(lane, pos, kSibCs);
                }
            } else if (GM_GEN_CACHE && SIB && l + 1 == (int)P.gen_level) {
                generate_cached<D>(P, S, scr, l + 1, F, lane, wacc);
            } else {
                generate<D>(P, S, l + 1, F, lane, wacc);
            }
            if (GM_GEN_CACHE && SIB && l + 2 == (int)P.gen_level) gen_prep<D>(P, S, scr, F, lane, wacc);
            if (SIB && l + 2 == (int)sibL) S.sibn[lane] = 0;        // new parents of level sib-1
            if (l + 1 == (int)P.par_level) prep_checks<D, SIB>(P, S, scr, l + 1, F, lane);
            if (!ENUM && bulk_two && l + 1 == last - 2) prep_two<D>(P, S, scr, l + 1, F, lane, wacc);
            if (!ENUM && bulk_last && l + 1 == last - 1) prep_last<D>(P, S, scr, l + 1, F, lane, wacc);
            if (lane == 0) { S.ci[l + 1] = 0; S.cj[l + 1] = 0; }
            __syncwarp();
            ++l;
        }
        if (lane == 0) work_add(P, C, S.home, -1);
    }
    // flush counters
    GM_ADD_WORDS(wacc);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        add_count(my_count, __shfl_xor_sync(FULL, my_count, o), ovf);
        my_tasks += __shfl_xor_sync(FULL, my_tasks, o);
        my_words += __shfl_xor_sync(FULL, my_words, o);
    }
    ovf = __any_sync(FULL, ovf);
    if (lane == 0) {
        if (ovf) atomicExch(&C->overflow, 1);
        if (my_count) {
            const unsigned long long old = atomicAdd(&C->count, my_count);
            if (old + my_count < old) atomicExch(&C->overflow, 1);
        }
        atomicAdd(&C->tasks, my_tasks);
        atomicAdd(&C->words, my_words);
        atomicAdd(&C->rounds, my_rounds);
        if (my_don) atomicAdd(&C->donations, my_don);
    }
}

// ------------------------------------------------------------------ BFS expansion

// One warp per partial match of depth d (level-major input).  MODE 0: count children
// into *ctr (and, if item_off, each item's child count into item_off[item]).  MODE 1: write
// children (depth d+1, level-major, stride out_stride) -- at item_off[item] + rank within the
// item when item_off is given (the exclusive scan of MODE 0's counts: a deterministic pool,
// identical on every rank), else at atomically claimed positions.  MODE 2: write children
// as final enumerate rows (by query-vertex column).
template <int MODE>
__global__ void __launch_bounds__(256) k_expand(const SearchParams P, const uint32_t *__restrict__ in,
                                                unsigned long long nin, uint32_t d, uint32_t *__restrict__ outp,
                                                unsigned long long out_stride, unsigned long long out_cap,
                                                unsigned long long *__restrict__ ctr,
                                                unsigned long long *__restrict__ item_off) {
    const uint32_t lane = threadIdx.x & 31;
    const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const uint32_t bw = P.bw[d], lab = P.lab[d];
    unsigned long long local = 0;
    uint32_t scratch = 0;   // word counter (unused: the BFS phase is not part of the DFS roofline)
    for (unsigned long long it = warp; it < nin; it += nwarps) {
        const uint32_t m = lane < d ? in[(unsigned long long)lane * nin + it] : 0;
        uint32_t lo = 0, hi = 0, len = 0xffffffffu;
        if (lane < d && ((bw >> lane) & 1u)) {
            const uint32_t row = m * P.S + lab;
            lo = ld_nc(P.offs + row); hi = ld_nc(P.offs + row + 1); len = hi - lo;
        }
        // source = backward neighbour with the shortest slice (ties: deepest level)
        uint32_t best = len, bl = lane;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint32_t ob = __shfl_xor_sync(FULL, best, o), oll = __shfl_xor_sync(FULL, bl, o);
            if (ob < best || (ob == best && oll > bl)) { best = ob; bl = oll; }
        }
        uint32_t cb = __shfl_sync(FULL, lo, bl);
        const uint32_t checks = bw & ~(1u << bl);
        {   // symmetry breaking: cut the sorted slice to [lb, ub) (see generate)
            const uint32_t gtm = P.sb_gt[d], ltm = P.sb_lt[d];
            if (gtm | ltm) {
                uint32_t lb = (lane < d && ((gtm >> lane) & 1u)) ? m + 1 : 0u;
                uint32_t ub = (lane < d && ((ltm >> lane) & 1u)) ? m : 0xffffffffu;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    lb = max(lb, __shfl_xor_sync(FULL, lb, o));
                    ub = min(ub, __shfl_xor_sync(FULL, ub, o));
                }
                uint32_t a = 0, e = best;
                if (lane == 0 && best) {
                    if (lb > 0) a = lower_bound_idx(P.nbr + cb, best, lb, scratch);
                    if (ub != 0xffffffffu) e = lower_bound_idx(P.nbr + cb, best, ub, scratch);
                }
                a = __shfl_sync(FULL, a, 0);
                e = __shfl_sync(FULL, e, 0);
                cb += a;
                best = e > a ? e - a : 0;
            }
        }
        unsigned long long item_base = 0, item_cnt = 0;
        if (MODE == 1 && item_off) item_base = item_off[it];
        for (uint32_t j0 = 0; j0 < best; j0 += 32) {
            const uint32_t j = j0 + lane;
            bool F = j < best;
            const uint32_t v = F ? ld_nc(P.nbr + cb + j) : 0;
            if (F) F = cand_bit(P, d, v, scratch);
            const uint32_t gt = P.sb_gt[d], lt = P.sb_lt[d];
            for (uint32_t i = 0; i < d; ++i) {
                const uint32_t mi = __shfl_sync(FULL, m, i);
                if (F && v == mi) F = false;
                if (F && ((gt >> i) & 1u) && !(v > mi)) F = false;      // symmetry breaking
                if (F && ((lt >> i) & 1u) && !(v < mi)) F = false;
                if (F && ((checks >> i) & 1u)) F = has_edge(P, mi, P.lab[i], v, lab, scratch);
            }
            const uint32_t fm = __ballot_sync(FULL, F);
            if (MODE == 0) {
                local += __popc(fm);
                item_cnt += __popc(fm);
            } else if (fm) {
                unsigned long long basepos = 0;
                if (MODE == 1 && item_off) {
                    basepos = item_base + item_cnt;
                    item_cnt += __popc(fm);
                } else {
                    if (lane == 0) basepos = atomicAdd(ctr, (unsigned long long)__popc(fm));
                    basepos = __shfl_sync(FULL, basepos, 0);
                }
                const unsigned long long pos = basepos + __popc(fm & ((1u << lane) - 1));
                const bool wr = F && pos < out_cap;
                for (uint32_t i = 0; i < d; ++i) {
                    const uint32_t mi = __shfl_sync(FULL, m, i);
                    if (wr) {
                        if (MODE == 1) outp[i * out_stride + pos] = mi;
                        else outp[pos * P.nq + P.col[i]] = ld_nc(P.new2old + mi);
                    }
                }
                if (wr) {
                    if (MODE == 1) outp[d * out_stride + pos] = v;
                    else outp[pos * P.nq + P.col[d]] = ld_nc(P.new2old + v);
                }
            }
        }
        if (MODE == 0 && item_off && lane == 0) item_off[it] = item_cnt;
    }
    if (MODE == 0 && lane == 0 && local) atomicAdd(ctr, local);
}

// Root candidates owned by this rank: cand bit of phi[0] set and (o / chunk) % world == rank
// for the ORIGINAL id o (ownership is defined on the caller's ids; device ids are degree-
// ordered and would put all hubs on one rank).  User roots arrive as original ids.
// Selected with a stable device-wide select, so the root list -- and the BFS pool built
// from it -- is identical run to run and rank to rank (needed by the shared pool counter).
struct RootSel {
    const uint32_t *cand, *vlab, *new2old, *old2new, *user;
    unsigned long long n;
    uint32_t candoff, lab0, rank, world, chunk;
    __device__ uint32_t operator()(unsigned long long i) const {
        const unsigned long long o = user ? user[i] : new2old[i];
        if (o >= n || (o / chunk) % world != rank) return 0xffffffffu;
        const uint32_t v = user ? old2new[o] : (uint32_t)i;
        if (vlab[v] != lab0 || !((cand[candoff + (v >> 5)] >> (v & 31)) & 1u)) return 0xffffffffu;
        return v;
    }
};
// Seeded permutation key of a root (splitmix64 finaliser of seed and vertex): sorting the
// root list by it gives a pseudo-random root order (gm_run_opts.root_seed).
struct RootKey {
    const uint32_t *roots;
    unsigned long long seed;
    __device__ unsigned long long operator()(unsigned long long i) const {
        unsigned long long z = seed * 0x9E3779B97F4A7C15ull + roots[i] + 1;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
};
__global__ void k_root_keys(RootKey rk, unsigned long long n, unsigned long long *keys) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        keys[i] = rk(i);
}
struct NotNone {
    __device__ bool operator()(uint32_t x) const { return x != 0xffffffffu; }
};

__global__ void k_write_single(const uint32_t *__restrict__ roots, unsigned long long n, uint32_t *__restrict__ out,
                               unsigned long long cap, const uint32_t *__restrict__ new2old) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n && i < cap;
         i += (unsigned long long)gridDim.x * blockDim.x)
        out[i] = new2old[roots[i]];
}


__global__ void k_init_ring(unsigned long long *seq, unsigned long long cap) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < cap;
         i += (unsigned long long)gridDim.x * blockDim.x)
        seq[i] = i;
}

// ------------------------------------------------------------------ host orchestration

struct Workspace {
    Ctrl *ctrl = nullptr;
    uint32_t *q_items = nullptr;
    unsigned long long *q_seq = nullptr;
    unsigned long long q_cap = 0;
    uint32_t *buf[2] = {nullptr, nullptr};
    size_t buf_bytes[2] = {0, 0};
    uint32_t *tmp = nullptr;        // CUB scratch
    size_t tmp_bytes = 0;
    uint32_t *item_off = nullptr;   // per-item child counts / offsets of a BFS level (u64)
    size_t item_off_bytes = 0;
    uint32_t *sib = nullptr;        // sibling-prefix buffers (every warp a grid can hold)
    size_t sib_bytes = 0;
    int sms = 148;
    ~Workspace() {
        cudaFree(ctrl); cudaFree(q_items); cudaFree(q_seq); cudaFree(buf[0]); cudaFree(buf[1]);
        cudaFree(tmp); cudaFree(item_off); cudaFree(sib);
    }
};

static int ensure(uint32_t *&p, size_t &have, size_t need) {
    if (have >= need) return GM_OK;
    cudaFree(p);
    p = nullptr;
    have = 0;
    size_t want = need + need / 4;
    GM_CK(cudaMalloc(&p, want));
    have = want;
    return GM_OK;
}

// shared memory of a warp's stack with `levels` levels allocated
template <int D>
static size_t stack_bytes(uint32_t levels) {
    // lv is the last member and every Level is a multiple of 16 bytes: the header is the rest
    using L = typename WarpStack<D>::Level;
    static_assert(sizeof(L) % 16 == 0, "stack levels keep 16-byte alignment");
    return sizeof(WarpStack<D>) - sizeof(L) * D + sizeof(L) * levels;
}

template <int D, bool ENUM, bool WORDS, int MODE>
static int launch_dfs(SearchParams P, int sms, uint32_t wpb, uint32_t bps, uint32_t sharers, cudaStream_t st,
                      uint32_t *grid_out, uint32_t *block_out) {
    // levels: at most D (a query of nq <= D vertices, its counted last levels not stored)
    P.levels = std::min<uint32_t>(P.levels ? P.levels : (uint32_t)D, (uint32_t)D);
    P.stack_bytes = (uint32_t)stack_bytes<D>(P.levels);
    P.aux_row = P.rows_chk + P.rows_last + P.rows_gen;
    P.warp_stride = (uint32_t)(P.stack_bytes + 128ull * (P.aux_row + P.rows_aux));
    auto kern = k_dfs<D, ENUM, WORDS, MODE>;
    constexpr uint32_t wmax = dfs_max_warps<D>();
    GM_REQ(wpb <= wmax, GM_ERR_ARG, "warps_per_block %u > %u (k_dfs<%d> launch bounds)", wpb, wmax, D);
    GM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::min<size_t>((size_t)P.warp_stride * (wpb ? wpb : wmax), 227u * 1024u)));
    // resident blocks for w warps per block (0 when a block does not fit)
    auto fit_for = [&](uint32_t w) -> int {
        if ((size_t)P.warp_stride * w > 227u * 1024u) return 0;
        int f = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f, kern, (int)(w * 32), (size_t)P.warp_stride * w) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        return f;
    };
    if (!wpb) {   // the block size with the most resident warps (ties: the larger block)
        uint32_t best = 0;
        for (uint32_t w = 1; w <= wmax; ++w) {
            const int f = fit_for(w);
            if (f > 0 && (uint32_t)f * w >= best) { best = (uint32_t)f * w; wpb = w; }
        }
        GM_REQ(best > 0, GM_ERR_LIMIT, "k_dfs: no block fits (%u B of shared memory per warp)", P.warp_stride);
    }
    const size_t smem = (size_t)P.warp_stride * wpb;
    const int fit = fit_for(wpb);
    GM_REQ(fit > 0, GM_ERR_LIMIT, "k_dfs: no block fits (smem %zu)", smem);
    const int per = bps ? std::min<int>((int)bps, fit) : fit;
    const uint32_t grid = (uint32_t)(sms * per);
    static const bool dbg = getenv("GM_DEBUG_LAUNCH") != nullptr;
    if (dbg)
        fprintf(stderr, "[gm] k_dfs<%d,%d,%d,%d> stack %zu B + %u scratch rows = %u B/warp, %u warps/block, "
                "%d blocks/SM fit, %d launched\n", D, (int)ENUM, (int)WORDS, MODE, (size_t)P.stack_bytes,
                P.aux_row + P.rows_aux, P.warp_stride, wpb, fit, per);
    // pool items per fetch: 32 (a full warp of parent lanes) when the pool is large; fewer
    // when it is small, so that every warp gets some initial work (§4.3).
    const unsigned long long nwarps = (unsigned long long)grid * wpb;
    // with a pool counter shared by `sharers` ranks, all of their warps draw from this pool
    const unsigned long long per_warp = P.pool_size / (4 * nwarps * std::max<uint32_t>(1, sharers));
    P.batch = (uint32_t)std::max<unsigned long long>(1, std::min<unsigned long long>(32, per_warp));
    kern<<<grid, wpb * 32, smem, st>>>(P);
    GM_CK(cudaGetLastError());
    *grid_out = grid;
    *block_out = wpb * 32;
    return GM_OK;
}

static int grid_for(unsigned long long work_items, int per_block, int sms) {
    unsigned long long g = (work_items + per_block - 1) / per_block;
    unsigned long long cap = (unsigned long long)sms * 16;
    if (g > cap) g = cap;
    return (int)(g ? g : 1);
}

}  // namespace gm

using namespace gm;

// Per-device search workspace (control block, steal ring, BFS pool buffers), created on
// first use and reused by every later search on that device, so that steady-state
// queries allocate nothing.  Searches on one device are serialised by its mutex.
struct DeviceWorkspace {
    std::mutex mu;
    Workspace *ws = nullptr;
};
static DeviceWorkspace g_ws[64];

static Workspace *device_workspace(int dev) {
    DeviceWorkspace &d = g_ws[dev & 63];
    if (!d.ws) {
        d.ws = new Workspace();
        cudaDeviceGetAttribute(&d.ws->sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return d.ws;
}

static int workspace_alloc_ring(Workspace &W) {
    if (!W.ctrl) GM_CK(cudaMalloc(&W.ctrl, sizeof(Ctrl)));
    if (!W.q_items) {
        W.q_cap = 1u << 18;
        GM_CK(cudaMalloc(&W.q_items, sizeof(uint32_t) * (size_t)W.q_cap * kItemWords));
        GM_CK(cudaMalloc(&W.q_seq, sizeof(unsigned long long) * (size_t)W.q_cap));
    }
    return GM_OK;
}

// A stealing team: every rank's control block and steal ring, mapped into this process.
struct gm_team {
    uint32_t n = 0, rank = 0;
    int dev = 0;
    uint32_t epoch = 0;      // searches run with this team so far (the same sequence on every rank)
    Ctrl *ctrl[kMaxTeam] = {};
    uint32_t *items[kMaxTeam] = {};
    unsigned long long *seq[kMaxTeam] = {};
};

extern "C" void gm_default_opts(gm_run_opts *o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->tau = 1000000;
    o->world = 1;
    o->root_chunk = 64;
    o->steal = 1;
    o->warps_per_block = 0;       // per query: the most resident warps
    o->pool_bytes_max = 1ull << 30;
}

// Query-vertex bitmask (by query vertex id) of phi[0..l-1].
static uint32_t backward_vertices(const gm_plan *p, uint32_t l) {
    uint32_t m = 0;
    for (uint32_t i = 0; i < l; ++i) m |= 1u << p->order[i];
    return m;
}

static int run_search(const gm_plan *p, const gm_run_opts *opts_in, bool enumerate, uint32_t *out, uint64_t cap,
                      int mem, uint64_t *count_out, int count_mem, gm_run_stats *stats, cudaStream_t st) {
    set_error("");
    GM_REQ(p && p->g, GM_ERR_ARG, "gm_count: NULL plan");
    GM_REQ(count_out, GM_ERR_ARG, "gm_count: NULL count_out");
    GM_REQ(mem == GM_MEM_HOST || mem == GM_MEM_DEVICE, GM_ERR_ARG, "bad mem");
    GM_REQ(count_mem == GM_MEM_HOST || count_mem == GM_MEM_DEVICE, GM_ERR_ARG, "bad mem");
    gm_run_opts o;
    gm_default_opts(&o);
    if (opts_in) {
        o = *opts_in;
        if (!o.tau) o.tau = 1000000;
        if (!o.world) o.world = 1;
        if (!o.root_chunk) o.root_chunk = 64;
        if (!o.pool_bytes_max) o.pool_bytes_max = 1ull << 30;
    }
    GM_REQ(o.rank < o.world, GM_ERR_ARG, "rank %u >= world %u", o.rank, o.world);
    GM_REQ(o.warps_per_block <= kDfsMaxWarps, GM_ERR_ARG, "warps_per_block %u > %u (k_dfs launch bounds)",
           o.warps_per_block, kDfsMaxWarps);
    GM_REQ(o.num_roots == 0 || o.roots, GM_ERR_ARG, "num_roots > 0 but roots NULL");
    GM_REQ(!o.team || (o.steal && o.shared_pool_ctr), GM_ERR_ARG,
           "a stealing team needs steal = 1 and a shared pool counter (every rank builds the same pool)");
    GM_REQ(!(o.flags & GM_FLAG_NO_POOL) || o.steal, GM_ERR_ARG, "GM_FLAG_NO_POOL needs steal = 1");
    const gm_graph *g = p->g;
    int dev = 0;
    GM_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_ws[dev & 63].mu);
    Workspace &W = *device_workspace(dev);
    gm_run_stats rs;
    memset(&rs, 0, sizeof(rs));
    uint32_t launches = 0;

    // every early return (GM_CK / GM_REQ) releases what this call created
    cudaEvent_t e0 = nullptr, e1 = nullptr, d0e = nullptr, d1e = nullptr;
    uint32_t *d_user = nullptr, *enum_dev = nullptr;
    struct Release {
        cudaEvent_t *ev[4];
        uint32_t **buf[2];
        ~Release() {
            for (auto e : ev) if (*e) cudaEventDestroy(*e);
            for (auto b : buf) if (*b) cudaFree(*b);
        }
    } release{{&e0, &e1, &d0e, &d1e}, {&d_user, &enum_dev}};
    GM_CK(cudaEventCreate(&e0)); GM_CK(cudaEventCreate(&e1));
    GM_CK(cudaEventCreate(&d0e)); GM_CK(cudaEventCreate(&d1e));
    GM_CK(cudaEventRecord(e0, st));

    // symmetry breaking (count only): embeddings satisfying the plan's conditions, times |Aut(Q)|.
    // Not with a user root list: "embeddings whose root is in the list" is not a union of
    // Aut(Q)-orbits.  (A rank partition is fine: every orbit representative has one root, so
    // the ranks' representative counts add up to the full one.)
    const bool use_sb = !enumerate && p->sb_ok && p->aut > 1 && !(o.flags & GM_FLAG_NO_SYMMETRY) && !o.roots;
    rs.automorphisms = use_sb ? p->aut : 1;

    // a stack level packs a slice length with its source level (GM_PACK_CS): lengths < 2^27
    GM_REQ(!GM_PACK_CS || g->dmax < (1u << 27), GM_ERR_LIMIT,
           "k_dfs: a vertex of degree %u (stack slices hold lengths < 2^27)", g->dmax);
    GM_REQ(!GM_PACK_PID || p->nq <= 8 || g->n < (1ull << 27), GM_ERR_LIMIT,
           "k_dfs: %llu vertices (queries of > 8 vertices: stack entries hold vertex ids < 2^27)",
           (unsigned long long)g->n);
    SearchParams P;
    memset(&P, 0, sizeof(P));
    P.offs = g->offs; P.nbr = g->nbr; P.cand = p->cand;
    P.S = g->S; P.nq = p->nq; P.words = p->words; P.use_cand = 1;
    for (uint32_t l = 0; l < p->nq; ++l) {
        P.lab[l] = p->qlab[p->order[l]] < g->S ? p->qlab[p->order[l]] : 0xfffffffeu;
        P.bw[l] = p->bw[l];
        P.candoff[l] = p->order[l] * p->words;
        // LDF/NLF count neighbours of u by label; if ALL of u's query neighbours precede it in
        // phi, a candidate adjacent to their (distinct, label-matching) images already meets
        // both bounds, so the bitmap test is implied and skipped (level 0 always tests).
        // With GM_FILTER_NONE the bitmap is the label test, implied by the label-partitioned slice.
        if (l == 0 || (p->filter != GM_FILTER_NONE && (p->qadj[p->order[l]] & ~backward_vertices(p, l)) != 0))
            P.cand_needed |= 1u << l;
        for (uint32_t i = 0; i < l; ++i)
            if (p->qlab[p->order[i]] == p->qlab[p->order[l]]) P.same_lab[l] |= 1u << i;
        if (use_sb) { P.sb_gt[l] = p->sb_gt[l]; P.sb_lt[l] = p->sb_lt[l]; }
        const uint32_t need = P.same_lab[l] | p->bw[l] | P.sb_gt[l] | P.sb_lt[l];
        P.walk_low[l] = need ? (uint32_t)__builtin_ctz(need) : l;
        P.col[l] = p->order[l];
    }
    P.nhubs = g->nhubs;
    P.hub_bits = g->hub_bits;
    P.hub_words = g->hub_words;
    P.hub_summ = g->hub_summ;
    P.summ_words = g->summ_words;
    P.summ_first = g->summ_first;
    P.new2old = g->new2old;
    P.old2new = g->old2new;
    if (!W.ctrl) GM_CK(cudaMalloc(&W.ctrl, sizeof(Ctrl)));
    GM_CK(cudaMemsetAsync(W.ctrl, 0, sizeof(Ctrl), st));
    P.ctrl = W.ctrl;
    unsigned long long *ctr_count = &W.ctrl->count;
    unsigned long long *ctr_aux = &W.ctrl->out_ctr;

    // ---- root candidates (rank share)
    // a non-NULL root list restricts phi[0]'s images to it (an empty list: no embeddings)
    const unsigned long long nroot_cap = o.roots ? o.num_roots : g->n;
    int rc = ensure(W.buf[0], W.buf_bytes[0], sizeof(uint32_t) * (nroot_cap ? nroot_cap : 1));
    if (rc) return rc;
    if (o.num_roots) {
        GM_CK(cudaMalloc(&d_user, sizeof(uint32_t) * o.num_roots));
        GM_CK(cudaMemcpyAsync(d_user, o.roots, sizeof(uint32_t) * o.num_roots, cudaMemcpyHostToDevice, st));
    }
    if (nroot_cap) {
        RootSel sel;
        sel.cand = p->cand; sel.vlab = g->lab; sel.new2old = g->new2old; sel.old2new = g->old2new;
        sel.user = d_user; sel.n = g->n; sel.candoff = P.candoff[0]; sel.lab0 = P.lab[0];
        // with a shared pool counter every rank builds the SAME (whole) pool
        sel.rank = o.shared_pool_ctr ? 0 : o.rank;
        sel.world = o.shared_pool_ctr ? 1 : o.world;
        sel.chunk = o.root_chunk;
        auto items = thrust::make_transform_iterator(thrust::counting_iterator<unsigned long long>(0), sel);
        size_t tb = 0;
        GM_CK(cub::DeviceSelect::If(nullptr, tb, items, W.buf[0], ctr_aux, (int64_t)nroot_cap, NotNone(), st));
        rc = ensure(W.tmp, W.tmp_bytes, tb + 16);
        if (rc) return rc;
        GM_CK(cub::DeviceSelect::If(W.tmp, tb, items, W.buf[0], ctr_aux, (int64_t)nroot_cap, NotNone(), st));
        launches += 1;
    }
    unsigned long long nroots = 0;
    GM_CK(cudaMemcpyAsync(&nroots, ctr_aux, sizeof(nroots), cudaMemcpyDeviceToHost, st));
    GM_CK(cudaStreamSynchronize(st));
    if (d_user) { cudaFree(d_user); d_user = nullptr; }
    rs.roots = nroots;
    if (o.root_seed && nroots > 1) {
        // seeded root order: sort (key, root) pairs by the key; buf[1] holds keys in/out and
        // roots out, item_off the keys' sorted copy
        const size_t kb = sizeof(unsigned long long) * nroots;
        rc = ensure(W.buf[1], W.buf_bytes[1], 2 * kb + sizeof(uint32_t) * nroots);
        if (rc) return rc;
        rc = ensure(W.item_off, W.item_off_bytes, kb);
        if (rc) return rc;
        unsigned long long *keys = reinterpret_cast<unsigned long long *>(W.buf[1]);
        unsigned long long *keys_out = reinterpret_cast<unsigned long long *>(W.item_off);
        uint32_t *roots_out = reinterpret_cast<uint32_t *>(keys + nroots);
        k_root_keys<<<grid_for(nroots, 256, W.sms), 256, 0, st>>>(RootKey{W.buf[0], o.root_seed}, nroots, keys);
        GM_CK(cudaGetLastError());
        size_t tb = 0;
        GM_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_out, W.buf[0], roots_out, (int64_t)nroots, 0, 64, st));
        rc = ensure(W.tmp, W.tmp_bytes, tb + 16);
        if (rc) return rc;
        GM_CK(cub::DeviceRadixSort::SortPairs(W.tmp, tb, keys, keys_out, W.buf[0], roots_out, (int64_t)nroots, 0, 64, st));
        GM_CK(cudaMemcpyAsync(W.buf[0], roots_out, sizeof(uint32_t) * nroots, cudaMemcpyDeviceToDevice, st));
        launches += 2;
    }

    uint32_t *frontier = W.buf[0];
    int cur = 0;
    unsigned long long P_n = nroots;
    uint32_t d = 1;
    unsigned long long total = 0;
    bool done = false, overflow = false;
    unsigned long long zero = 0;

    // enum_dev: device staging for host-side enumerate output (released by `release`;
    // copied to `out` once, at the end)
    if (enumerate && mem != GM_MEM_DEVICE && cap) {
        if (cudaMalloc(&enum_dev, sizeof(uint32_t) * cap * p->nq) != cudaSuccess) {
            cudaGetLastError();
            enum_dev = nullptr;
            set_error("gm_enumerate: cannot stage %llu rows on the device", (unsigned long long)cap);
            return GM_ERR_NOMEM;
        }
    }
    auto out_dev = [&]() -> uint32_t * { return mem == GM_MEM_DEVICE ? out : enum_dev; };

    if (p->nq == 1) {
        total = nroots;
        if (enumerate && nroots && cap) {
            k_write_single<<<grid_for(nroots, 256, W.sms), 256, 0, st>>>(frontier, nroots, out_dev(), cap, g->new2old);
            GM_CK(cudaGetLastError());
            ++launches;
        }
        done = true;
    }

    // a query vertex without candidates (e.g. a label absent from G): no embeddings, and the
    // search kernels never see a label outside [0, S)
    for (uint32_t u = 0; u < p->nq && !done; ++u)
        if (p->cand_count[u] == 0) { total = 0; done = true; }

    // ---- initialization phase: BFS to tau partial matches (§4.3)
    while (!done) {
        if (P_n == 0) { total = 0; done = true; break; }
        if (P_n >= o.tau) break;
        GM_CK(cudaMemcpyAsync(ctr_count, &zero, sizeof(zero), cudaMemcpyHostToDevice, st));
        const int gb = grid_for(P_n * 32, 256, W.sms);
        const bool last_level = d + 1 == p->nq;
        unsigned long long *item_off = nullptr;
        if (!last_level) {   // per-item counts -> offsets: a deterministic next level
            rc = ensure(W.item_off, W.item_off_bytes, sizeof(unsigned long long) * P_n);
            if (rc) return rc;
            item_off = reinterpret_cast<unsigned long long *>(W.item_off);
        }
        k_expand<0><<<gb, 256, 0, st>>>(P, frontier, P_n, d, nullptr, 0, 0, ctr_count, item_off);
        GM_CK(cudaGetLastError());
        ++launches;
        unsigned long long c = 0;
        GM_CK(cudaMemcpyAsync(&c, ctr_count, sizeof(c), cudaMemcpyDeviceToHost, st));
        GM_CK(cudaStreamSynchronize(st));
        if (d + 1 == p->nq) {
            total = c;
            if (enumerate && c && cap) {
                GM_CK(cudaMemcpyAsync(ctr_aux, &zero, sizeof(zero), cudaMemcpyHostToDevice, st));
                k_expand<2><<<gb, 256, 0, st>>>(P, frontier, P_n, d, out_dev(), 0, cap, ctr_aux, nullptr);
                GM_CK(cudaGetLastError());
                ++launches;
            }
            done = true;
            break;
        }
        const size_t need = sizeof(uint32_t) * (size_t)c * (d + 1);
        if (c == 0) { total = 0; done = true; break; }
        if (need > o.pool_bytes_max) break;
        rc = ensure(W.buf[cur ^ 1], W.buf_bytes[cur ^ 1], need);
        if (rc) return rc;
        {   // exclusive scan of the per-item counts (in place)
            size_t tb = 0;
            GM_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, item_off, item_off, (int64_t)P_n, st));
            rc = ensure(W.tmp, W.tmp_bytes, tb + 16);
            if (rc) return rc;
            GM_CK(cub::DeviceScan::ExclusiveSum(W.tmp, tb, item_off, item_off, (int64_t)P_n, st));
            ++launches;
        }
        k_expand<1><<<gb, 256, 0, st>>>(P, frontier, P_n, d, W.buf[cur ^ 1], c, c, ctr_aux, item_off);
        GM_CK(cudaGetLastError());
        ++launches;
        cur ^= 1;
        frontier = W.buf[cur];
        P_n = c;
        ++d;
    }
    rs.pool_size = P_n;
    rs.pool_depth = d;

    // ---- DFS (fine-grained, batch exploration, stealing)
    if (!done) {
        if (o.steal) {
            rc = workspace_alloc_ring(W);
            if (rc) return rc;
        }
        if (o.steal) {
            k_init_ring<<<grid_for(W.q_cap, 256, W.sms), 256, 0, st>>>(W.q_seq, W.q_cap);
            GM_CK(cudaGetLastError());
            ++launches;
        }
        GM_CK(cudaMemsetAsync(W.ctrl, 0, sizeof(Ctrl), st));
        P.pool = frontier;
        P.pool_ctr = o.shared_pool_ctr ? reinterpret_cast<unsigned long long *>(o.shared_pool_ctr)
                                       : &W.ctrl->pool_ctr;
        P.pool_sys = o.shared_pool_ctr ? 1u : 0u;
        P.pool_size = P_n;
        P.d0 = d;
        P.steal = o.steal ? 1 : 0;
        P.q_items = W.q_items; P.q_seq = W.q_seq; P.q_cap = o.steal ? W.q_cap : 1;
        P.no_pool = (o.flags & GM_FLAG_NO_POOL) ? 1u : 0u;
        if (o.team) {
            gm_team *t = o.team;
            GM_REQ(t->dev == dev && t->ctrl[t->rank] == W.ctrl && t->items[t->rank] == W.q_items,
                   GM_ERR_ARG, "gm_run_opts.team was opened on another device or process state");
            P.team_n = t->n;
            P.team_rank = t->rank;
            P.epoch = ++t->epoch;
            // this rank's lineage word for the new search: (epoch << 32) | 0, published before
            // the DFS launch (the control block was just zeroed)
            const unsigned long long tw = (unsigned long long)P.epoch << 32;
            GM_CK(cudaMemcpyAsync(&W.ctrl->tword, &tw, sizeof(tw), cudaMemcpyHostToDevice, st));
            for (uint32_t r = 0; r < t->n; ++r) {
                P.team_ctrl[r] = t->ctrl[r];
                P.team_items[r] = t->items[r];
                P.team_seq[r] = t->seq[r];
            }
        }
        if (enumerate) {
            P.out = out_dev(); P.out_cap = cap;
            P.stop_at_cap = (o.flags & GM_FLAG_STOP_AT_CAPACITY) ? 1u : 0u;
        }
        // the time limit covers the DFS launch (the BFS init phase is short and bounded by tau)
        P.limit_ns = o.time_limit_ms > 0 ? (unsigned long long)(o.time_limit_ms * 1e6) : 0ull;
        {   // last-level set counting applies when phi[last] has exactly one backward neighbour
            const uint32_t last = p->nq - 1, bwl = p->bw[last];
            if (!enumerate && !(o.flags & GM_FLAG_NO_SET_COUNT) && last >= 1 && __builtin_popcount(bwl) == 1) {
                const uint32_t b = (uint32_t)__builtin_ctz(bwl);
                P.bulk_last = 1;
                P.last_b = b;
                for (uint32_t i = 0; i < last; ++i) {
                    if (i != b && p->qlab[p->order[i]] == p->qlab[p->order[last]]) P.last_same |= 1u << i;
                    if ((p->qadj[p->order[b]] >> p->order[i]) & 1u) P.last_adj |= 1u << i;
                }
                const uint32_t l = last - 1;   // the level count_last runs at
                const uint32_t below = (1u << l) - 1;
                P.last_sb = (P.sb_gt[last] | P.sb_lt[last]) ? 1u : 0u;
                uint32_t need = (b < l ? 1u << b : 0u) | (P.last_same & ~P.last_adj & below);
                if (P.last_sb) need |= (P.last_same & P.last_adj & below) | ((P.sb_gt[last] | P.sb_lt[last]) & below);
                P.last_low = need ? (uint32_t)__builtin_ctz(need) : l;
                P.last_k = (uint32_t)__builtin_popcount(P.last_same & ~P.last_adj & below);
                P.last_ka = P.last_sb ? (uint32_t)__builtin_popcount(P.last_same & P.last_adj & below) : 0u;
                // The candidate-filter test of phi[last-1] is subsumed by the set count: its only
                // possible forward neighbour is phi[last], so a candidate the (sound) filter
                // rejects has no valid extension and count_last returns exactly 0 for it.
                // Skipping the test takes a dependent bitmap load off every task of the level.
                P.cand_needed &= ~(1u << l);
            }
        }
        {   // pair counting: phi[last-1], phi[last] each with one backward neighbour, not adjacent,
            // no symmetry-breaking bounds and no filter test on either (both are implied)
            const uint32_t last = p->nq - 1;
            if (P.bulk_last && last >= 2 && !(o.flags & GM_FLAG_NO_PAIR_COUNT) &&
                __builtin_popcount(p->bw[last - 1]) == 1 && !((p->bw[last] >> (last - 1)) & 1u) &&
                !(P.sb_gt[last] | P.sb_lt[last] | P.sb_gt[last - 1] | P.sb_lt[last - 1]) &&
                !((P.cand_needed >> (last - 1)) & 3u)) {
                const uint32_t b6 = (uint32_t)__builtin_ctz(p->bw[last - 1]), b7 = P.last_b;
                const uint32_t l = last - 2;
                P.bulk_two = 1;
                P.two_b6 = b6;
                P.two_b7 = b7;
                for (uint32_t i = 0; i <= l; ++i) {
                    const uint32_t ui = p->order[i];
                    if (i != b6 && p->qlab[ui] == p->qlab[p->order[last - 1]]) P.two_same6 |= 1u << i;
                    if (i != b7 && p->qlab[ui] == p->qlab[p->order[last]]) P.two_same7 |= 1u << i;
                    if ((p->qadj[p->order[b6]] >> ui) & 1u) P.two_adj6 |= 1u << i;
                    if ((p->qadj[p->order[b7]] >> ui) & 1u) P.two_adj7 |= 1u << i;
                }
                const uint32_t below = (1u << l) - 1;
                const uint32_t need = (b6 < l ? 1u << b6 : 0u) | (b7 < l ? 1u << b7 : 0u) |
                                      ((P.two_same6 | P.two_same7) & below);
                P.two_low = need ? (uint32_t)__builtin_ctz(need) : l;
                P.two_walk = ((b6 == l && (P.two_same6 & below)) || (b7 == l && (P.two_same7 & below))) ? 1u : 0u;
            }
        }
        {   // per-parent check lists at the level holding almost all tasks (prep_checks); none
            // with pair counting (its levels have no checks)
            const uint32_t last = p->nq - 1;
            P.par_level = P.bulk_two ? last - 2 : (P.bulk_last ? last - 1 : last);
            if (P.par_level != ~0u) {
                const uint32_t l = P.par_level;
                const uint32_t need = (p->bw[l] | P.same_lab[l]) & ((1u << l) - 1);
                P.par_low = need ? (uint32_t)__builtin_ctz(need) : l;
            }
        }
        {   // sibling prefixes (sib_append): phi[last] adjacent to phi[last-1] and to all of its
            // backward neighbours, same label, a filter no stricter (LDF: query degree, NLF:
            // neighbour counts per label, each >= phi[last-1]'s), bounds including M[phi[last]] <
            // M[phi[last-1]] and all of phi[last-1]'s; level last-1 searched by the DFS
            const uint32_t last = p->nq - 1;
            if (!enumerate && GM_SIB && !(o.flags & GM_FLAG_NO_SIBLING) && use_sb && last >= 2 && p->nq <= 8 &&
                P.par_level == last && d + 1 <= last) {
                const uint32_t a = p->order[last - 1], b = p->order[last];
                const uint32_t bwa = p->bw[last - 1], bwb = p->bw[last];
                bool ok = (bwb & bwa) == bwa && ((bwb >> (last - 1)) & 1u) && p->qlab[a] == p->qlab[b] &&
                          ((P.sb_lt[last] >> (last - 1)) & 1u) && !(P.sb_gt[last - 1] & ~P.sb_gt[last]) &&
                          !(P.sb_lt[last - 1] & ~P.sb_lt[last]);
                if (ok && p->filter >= GM_FILTER_LDF) ok = p->qdeg[a] <= p->qdeg[b];
                if (ok && p->filter >= GM_FILTER_NLF) {
                    for (uint32_t x = 0; x < p->nq && ok; ++x) {
                        const uint32_t L = p->qlab[x];
                        uint32_t ca = 0, cb2 = 0;
                        for (uint32_t y = 0; y < p->nq; ++y) {
                            if (p->qlab[y] != L) continue;
                            ca += (p->qadj[a] >> y) & 1u;
                            cb2 += (p->qadj[b] >> y) & 1u;
                        }
                        ok = ca <= cb2;
                    }
                }
                if (ok) {
                    // one buffer row set per warp a grid can hold (8-level kernels: <= 16 blocks of
                    // 4 warps per SM)
                    const size_t need = sizeof(uint32_t) * (size_t)W.sms * 16 * dfs_max_warps<8>() * 32 * kSibCap;
                    rc = ensure(W.sib, W.sib_bytes, need);
                    if (rc) return rc;
                    P.sib = W.sib;
                    P.sib_level = last;
                    P.sib_cap = kSibCap;
                    P.sib_chk = bwb & ~bwa;
                }
            }
        }
        {   // cached GenerateTask part at the hot level (gen_prep): when it has backward rows or
            // bounds from levels <= l-2 and no sibling prefixes
            // symmetry bounds (whose cut is the costly part: two binary searches per task) and a
            // backward row, both from levels <= l-2; 8-level count kernels (measured: it helps
            // the 5-cycle, +70 % embeddings in 5 s, and costs other queries)
            const uint32_t l = P.par_level;
            const uint32_t far = l != ~0u && l >= 2 ? (1u << (l - 1)) - 1 : 0u;
            if (GM_GEN_CACHE && !(o.flags & GM_FLAG_NO_GEN_CACHE) && !enumerate && p->nq <= 8 && !P.sib_level &&
                !P.bulk_last && !P.bulk_two &&
                far && (p->bw[l] & far) && ((P.sb_gt[l] | P.sb_lt[l]) & far)) {
                P.gen_level = l;
                P.rows_gen = 5;
            }
        }
        {   // scratch rows: the most check images any task (or a par-level parent) holds, and the
            // set / pair counting words
            const uint32_t last = p->nq - 1;
            uint32_t rc = 0;
            for (uint32_t l = 1; l <= last; ++l) rc = std::max<uint32_t>(rc, (uint32_t)__builtin_popcount(p->bw[l]) - 1);
            if (P.par_level != ~0u && P.par_level >= 1) {   // (level 0 is never entered by the DFS)
                const uint32_t l = P.par_level;
                rc = std::max<uint32_t>(rc, (uint32_t)__builtin_popcount(p->bw[l]) - 1 +
                                                (uint32_t)__builtin_popcount(P.same_lab[l] & ~p->bw[l] & ((1u << l) - 1)));
            }
            uint32_t rl = P.bulk_last ? P.last_k + P.last_ka : 0u;
            if (P.bulk_two) rl = std::max<uint32_t>(rl, 6u);
#if GM_TWO_STAGE
            // staging buffer for the pair-count intersection (same-label leaves, two parents)
            if (P.bulk_two && P.lab[p->nq - 2] == P.lab[p->nq - 1] && P.two_b6 != P.two_b7) {
                P.two_stage_row = rl;
                rl += kStageWords / 32;
            }
#endif
            P.rows_chk = rc;
            P.rows_last = rl;
        }
        rs.paths = (P.bulk_last ? GM_PATH_SET_COUNT : 0u) | (P.bulk_two ? GM_PATH_PAIR_COUNT : 0u) |
                   (P.par_level != ~0u && P.par_level >= d ? GM_PATH_PAR_CHECKS : 0u) |
                   (use_sb ? GM_PATH_SYMMETRY : 0u) | (P.sib_level ? GM_PATH_SIBLING : 0u) |
                   (P.gen_level ? GM_PATH_GEN_CACHE : 0u);
        // stack depth: the smallest instantiation that holds the query (17-24-vertex counts get
        // a 24-level stack: 11.6 KB per warp instead of 15.5, so more warps stay resident)
        rs.stack_levels = p->nq <= 8 ? 8u : (p->nq <= 16 ? 16u : ((!enumerate && GM_D24 && p->nq <= 24) ? 24u : 32u));
        GM_CK(cudaEventRecord(d0e, st));
        const uint32_t nq = p->nq;
        const bool cw = (o.flags & GM_FLAG_COUNT_WORDS) != 0;
        const uint32_t sharers = o.shared_pool_ctr ? o.world : 1u;
#define GM_LAUNCH(DD, EE, WW, MM) launch_dfs<DD, EE, WW, MM>(P, W.sms, o.warps_per_block, o.blocks_per_sm, sharers, st, &rs.grid, &rs.block)
#define GM_LAUNCH_M(DD, MM) (cw ? GM_LAUNCH(DD, false, true, MM) : GM_LAUNCH(DD, false, false, MM))
#define GM_LAUNCH_D(DD) (mode == kModePair ? GM_LAUNCH_M(DD, kModePair) : \
                         (mode == kModeSet ? GM_LAUNCH_M(DD, kModeSet) : GM_LAUNCH_M(DD, kModePlain)))
        // the smallest kernel that holds this query's paths (the enumerate kernels run every
        // level by tasks: no counting code)
        const int mode = (nq <= 8 && (P.sib_level || P.gen_level)) ? kModePat
                       : (P.bulk_two ? kModePair : (P.bulk_last ? kModeSet : kModePlain));
        {   // stack levels the search touches: the slice of level `top` is the deepest entry
            // written (a counted level -- set counting of the last, pair counting of the last
            // two -- is never entered; only the flags the launched kernel honours count)
            const bool eff_two = !enumerate && mode == kModePair && P.bulk_two;
            const bool eff_last = !enumerate && (mode == kModeSet || mode == kModePair) && P.bulk_last;
            const uint32_t last = nq - 1;
            uint32_t top = last;
            if (eff_two && P.d0 + 2 <= last) top = last - 2;
            else if (eff_last && P.d0 + 1 <= last) top = last - 1;
            P.levels = top + 1;
            // counting state rows: the kernels of these modes run prep_last / prep_two
            P.rows_aux = enumerate ? 0u : (mode == kModePair ? 4u : (mode == kModeSet ? 3u : 0u));
        }
        if (enumerate)   // (enumerate never counts words: its cost is the output)
            rc = nq <= 8 ? GM_LAUNCH(8, true, false, kModePlain)
                         : (nq <= 16 ? GM_LAUNCH(16, true, false, kModePlain) : GM_LAUNCH(32, true, false, kModePlain));
        else if (nq <= 8)
            rc = mode == kModePat ? GM_LAUNCH_M(8, kModePat) : GM_LAUNCH_D(8);
        else if (nq <= 16)
            rc = GM_LAUNCH_D(16);
#if GM_D24
        else if (nq <= 24)
            rc = GM_LAUNCH_D(24);
#endif
        else
            rc = GM_LAUNCH_D(32);
#undef GM_LAUNCH_D
#undef GM_LAUNCH_M
#undef GM_LAUNCH_WP
#undef GM_LAUNCH
        if (rc) return rc;
        ++launches;
        rs.dfs_launches = 1;
        GM_CK(cudaEventRecord(d1e, st));
        Ctrl h;
        GM_CK(cudaMemcpyAsync(&h, W.ctrl, sizeof(h), cudaMemcpyDeviceToHost, st));
        GM_CK(cudaStreamSynchronize(st));
        total = h.count;
        overflow = h.overflow != 0;
        rs.tasks = h.tasks;
        rs.words = h.words;
        rs.rounds = h.rounds;
        rs.donations = h.donations;
        rs.timed_out = h.abort ? 1 : 0;
        GM_CK(cudaEventElapsedTime(&rs.dfs_ms, d0e, d1e));
#ifdef GM_LEVEL_STATS
        {
            unsigned long long lt[32], lp[32];
            GM_CK(cudaMemcpyFromSymbol(lt, g_level_tasks, sizeof(lt)));
            GM_CK(cudaMemcpyFromSymbol(lp, g_level_pass, sizeof(lp)));
            fprintf(stderr, "[level stats] d0=%u bulk_last=%u:", d, P.bulk_last);
            for (uint32_t i = 0; i < p->nq; ++i) fprintf(stderr, " L%u %.3g/%.3g", i, (double)lt[i], (double)lp[i]);
            fprintf(stderr, "\n");
            memset(lt, 0, sizeof(lt));
            GM_CK(cudaMemcpyToSymbol(g_level_tasks, lt, sizeof(lt)));
            GM_CK(cudaMemcpyToSymbol(g_level_pass, lt, sizeof(lt)));
        }
#endif
    }
    if (use_sb && __builtin_mul_overflow(total, (unsigned long long)p->aut, &total))   // one per Aut(Q)-orbit
        overflow = true;
    if (overflow) total = ~0ull;
    // ---- outputs
    if (enumerate && mem == GM_MEM_HOST && enum_dev && cap) {
        const uint64_t rows = std::min<uint64_t>(cap, total);
        GM_CK(cudaMemcpyAsync(out, enum_dev, sizeof(uint32_t) * rows * p->nq, cudaMemcpyDeviceToHost, st));
    }
    if (count_mem == GM_MEM_DEVICE) {
        GM_CK(cudaMemcpyAsync(ctr_count, &total, sizeof(total), cudaMemcpyHostToDevice, st));
        GM_CK(cudaMemcpyAsync(count_out, ctr_count, sizeof(total), cudaMemcpyDeviceToDevice, st));
    } else {
        *count_out = total;
    }
    GM_CK(cudaEventRecord(e1, st));
    GM_CK(cudaStreamSynchronize(st));
    GM_CK(cudaEventElapsedTime(&rs.total_ms, e0, e1));
    rs.count = total;
    rs.kernel_launches = launches;
    if (stats) *stats = rs;
    if (overflow) {
        set_error("gm_count: the number of embeddings exceeds 2^64 - 1");
        return GM_ERR_LIMIT;
    }
    return rs.timed_out ? GM_TIMEOUT : GM_OK;
}

extern "C" int gm_count(const gm_plan *p, const gm_run_opts *opts, uint64_t *count_out, int mem,
                        gm_run_stats *stats, void *stream) {
    return run_search(p, opts, false, nullptr, 0, GM_MEM_DEVICE, count_out, mem, stats, (cudaStream_t)stream);
}

extern "C" int gm_enumerate(const gm_plan *p, const gm_run_opts *opts, uint32_t *out, uint64_t capacity, int mem,
                            uint64_t *count_host, gm_run_stats *stats, void *stream) {
    GM_REQ(capacity == 0 || out, GM_ERR_ARG, "gm_enumerate: out NULL with capacity > 0");
    return run_search(p, opts, true, out, capacity, mem, count_host, GM_MEM_HOST, stats, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ cross-GPU stealing team

extern "C" int gm_team_export(void *handle_out) {
    set_error("");
    GM_REQ(handle_out, GM_ERR_ARG, "gm_team_export: NULL handle_out");
    static_assert(3 * sizeof(cudaIpcMemHandle_t) <= GM_TEAM_HANDLE_BYTES, "team handle size");
    int dev = 0;
    GM_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_ws[dev & 63].mu);
    Workspace &W = *device_workspace(dev);
    int rc = workspace_alloc_ring(W);
    if (rc) return rc;
    cudaIpcMemHandle_t h[3];
    GM_CK(cudaIpcGetMemHandle(&h[0], W.ctrl));
    GM_CK(cudaIpcGetMemHandle(&h[1], W.q_items));
    GM_CK(cudaIpcGetMemHandle(&h[2], W.q_seq));
    memset(handle_out, 0, GM_TEAM_HANDLE_BYTES);
    memcpy(handle_out, h, sizeof(h));
    return GM_OK;
}

extern "C" int gm_team_open(uint32_t world, uint32_t rank, const void *handles, gm_team **out) {
    set_error("");
    GM_REQ(handles && out, GM_ERR_ARG, "gm_team_open: NULL argument");
    GM_REQ(world >= 1 && world <= kMaxTeam && rank < world, GM_ERR_ARG, "gm_team_open: world %u rank %u (max %u)",
           world, rank, kMaxTeam);
    int dev = 0;
    GM_CK(cudaGetDevice(&dev));
    Workspace *W = nullptr;
    {
        std::lock_guard<std::mutex> lock(g_ws[dev & 63].mu);
        W = device_workspace(dev);
        int rc = workspace_alloc_ring(*W);
        if (rc) return rc;
    }
    gm_team *t = new gm_team();
    t->n = world; t->rank = rank; t->dev = dev;
    const uint8_t *hb = static_cast<const uint8_t *>(handles);
    for (uint32_t r = 0; r < world; ++r) {
        if (r == rank) {
            t->ctrl[r] = W->ctrl; t->items[r] = W->q_items; t->seq[r] = W->q_seq;
            continue;
        }
        cudaIpcMemHandle_t h[3];
        memcpy(h, hb + (size_t)r * GM_TEAM_HANDLE_BYTES, sizeof(h));
        void *p[3] = {nullptr, nullptr, nullptr};
        cudaError_t e = cudaSuccess;
        for (int k = 0; k < 3 && e == cudaSuccess; ++k) e = cudaIpcOpenMemHandle(&p[k], h[k], cudaIpcMemLazyEnablePeerAccess);
        t->ctrl[r] = static_cast<Ctrl *>(p[0]);
        t->items[r] = static_cast<uint32_t *>(p[1]);
        t->seq[r] = static_cast<unsigned long long *>(p[2]);
        if (e != cudaSuccess) {
            gm_team_free(t);
            cudaGetLastError();
            set_error("gm_team_open: cudaIpcOpenMemHandle for rank %u: %s", r, cudaGetErrorString(e));
            return GM_ERR_CUDA;
        }
    }
    *out = t;
    return GM_OK;
}

extern "C" void gm_team_free(gm_team *t) {
    if (!t) return;
    for (uint32_t r = 0; r < t->n; ++r) {
        if (r == t->rank) continue;
        if (t->ctrl[r]) cudaIpcCloseMemHandle(t->ctrl[r]);
        if (t->items[r]) cudaIpcCloseMemHandle(t->items[r]);
        if (t->seq[r]) cudaIpcCloseMemHandle(t->seq[r]);
    }
    delete t;
}

// ------------------------------------------------------------------ multi-GPU pool counter

extern "C" int gm_pool_counter_create(uint32_t slots, void **counter_dev, void *ipc_handle_out) {
    set_error("");
    GM_REQ(counter_dev && ipc_handle_out, GM_ERR_ARG, "gm_pool_counter_create: NULL argument");
    GM_REQ(slots >= 1 && slots <= (1u << 20), GM_ERR_ARG, "gm_pool_counter_create: slots %u outside [1, 2^20]", slots);
    static_assert(sizeof(cudaIpcMemHandle_t) <= GM_IPC_HANDLE_BYTES, "IPC handle size");
    void *p = nullptr;
    const size_t bytes = (size_t)slots * GM_POOL_COUNTER_STRIDE;   // one 128-byte line per slot
    GM_CK(cudaMalloc(&p, bytes));
    GM_CK(cudaMemset(p, 0, bytes));
    cudaIpcMemHandle_t h;
    GM_CK(cudaIpcGetMemHandle(&h, p));
    memset(ipc_handle_out, 0, GM_IPC_HANDLE_BYTES);
    memcpy(ipc_handle_out, &h, sizeof(h));
    *counter_dev = p;
    return GM_OK;
}

extern "C" int gm_pool_counter_open(const void *ipc_handle, void **counter_dev) {
    set_error("");
    GM_REQ(counter_dev && ipc_handle, GM_ERR_ARG, "gm_pool_counter_open: NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    void *p = nullptr;
    GM_CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *counter_dev = p;
    return GM_OK;
}

extern "C" int gm_pool_counter_reset(void *counter_dev, uint32_t slots, void *stream) {
    set_error("");
    GM_REQ(counter_dev, GM_ERR_ARG, "gm_pool_counter_reset: NULL counter");
    GM_REQ(slots >= 1, GM_ERR_ARG, "gm_pool_counter_reset: slots = 0");
    GM_CK(cudaMemsetAsync(counter_dev, 0, (size_t)slots * GM_POOL_COUNTER_STRIDE, (cudaStream_t)stream));
    return GM_OK;
}

extern "C" int gm_pool_counter_close(void *counter_dev, int owner) {
    if (!counter_dev) return GM_OK;
    if (owner) GM_CK(cudaFree(counter_dev));
    else GM_CK(cudaIpcCloseMemHandle(counter_dev));
    return GM_OK;
}
