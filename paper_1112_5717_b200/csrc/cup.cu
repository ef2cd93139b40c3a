// cup.cu -- host driver of the device-resident CUP recursion.
//
// Follows the reference's row-halving recursion cup_rec (proj/src/factor.cpp:30-81)
// with the same split k = m/2 down to leaves of <= PB rows, but every
// rank-dependent extent (r1, column origins, widths) is a Dyn expression over
// the device-resident rank prefix rp[]: the host walks a STATIC skeleton and
// enqueues kernels without ever reading a rank back, so one factorization is a
// single host-sync-free launch sequence (captured once into a CUDA graph and
// replayed).  Deviations from the reference's data movement, all value-neutral:
//   * U rows are not shifted up at every level (factor.cpp:62-70); they stay in
//     their pivot rows and are gathered through rrp[] when used as the B
//     operand, then placed once at the end (compact_u_rows).
//   * sigma is kept as the transposition list ipiv[] (perm.cpp:21-26) and
//     composed on the host at the end (factor.cpp:78-79).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "cup.h"
#include "kernels.cuh"
#include "runtime.h"

namespace rl {

CupEngine::CupEngine(i32 m, i32 n, i64 lda, u32 p) : m_(m), n_(n), lda_(lda), p_(p) {
    f_ = make_fp(p);
    L_ = limbs_for(p);
    // dry run to size the GEMM workspaces
    dry_ = true;
    // tuning / test knobs of the tiled top level
    if (const char* e = getenv("RL_TILE_G")) tile_g_ = atoi(e);
    if (const char* e = getenv("RL_TILE_MIN_M")) tile_min_m_ = atoi(e);
    if (const char* e = getenv("RL_TILE_MAX_M")) tile_max_m_ = atoi(e);
    if (tile_g_ > 0) tile_g_ = std::max(PB, tile_g_ / PB * PB);  // whole leaves
    if (const char* e = getenv("RL_TILE_CTAS")) tile_ctas_ = atoi(e);
    if (const char* e = getenv("RL_TILE_AFTER_REST")) tile_after_rest_ = atoi(e) != 0;
    if (const char* e = getenv("RL_REST_PIECES")) rest_pieces_ = atoi(e) != 0;
    if (const char* e = getenv("RL_REST_SPLIT")) rest_split_ = atoi(e);
    if (const char* e = getenv("RL_S2_PRIO")) s2_prio_ = atoi(e) != 0;
    if (m_ > 0 && n_ > 0) {
        if (tiled_on()) tiled(tile_g_);
        else node(0, m_);
    }
    dry_ = false;
    const i32 k = std::min(m_, n_);
    // All per-factorization metadata (rank prefix, profile, transpositions, panel
    // scratch, leaf inverses, inverse table) in ONE allocation: the latency-bound
    // panel kernels touch all of it, and one mapping keeps their TLB footprint small.
    auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t o_rp = 0;
    const size_t o_rrp = o_rp + up(sizeof(i32) * (m_ + 1));
    const size_t o_ipiv = o_rrp + up(sizeof(i32) * (k + 1));
    const size_t o_ps = o_ipiv + up(sizeof(i32) * (k + 1));
    const size_t o_uinv = o_ps + up(sizeof(PanelScratch));
    const size_t o_flags = o_uinv + up(sizeof(u32) * PB * PB * (leaf_of_.size() + 1));
    const size_t o_uready = o_flags + up(sizeof(i32) * (leaf_of_.size() + 1));
    const size_t o_tab = o_uready + up(sizeof(i32) * (leaf_of_.size() + 2));
    const size_t o_ninv = o_tab + up(p_ <= 65536u ? 65536 * sizeof(uint16_t) : 0);
    const size_t total = o_ninv + sizeof(u32) * NINV_LD * NINV_LD * ninv_slot_.size();
    RL_CUDA_CHECK(cudaMalloc(&meta_, total));
    char* base = static_cast<char*>(meta_);
    rp_ = reinterpret_cast<i32*>(base + o_rp);
    rrp_ = reinterpret_cast<i32*>(base + o_rrp);
    ipiv_ = reinterpret_cast<i32*>(base + o_ipiv);
    ps_ = reinterpret_cast<PanelScratch*>(base + o_ps);
    // set-up work on a private non-blocking stream: nothing here touches the
    // legacy stream (another host thread may be capturing a graph meanwhile)
    cudaStream_t init_s = nullptr;
    RL_CUDA_CHECK(cudaStreamCreateWithFlags(&init_s, cudaStreamNonBlocking));
    RL_CUDA_CHECK(cudaMemsetAsync(ps_, 0, sizeof(PanelScratch), init_s));
    uinv_ = reinterpret_cast<u32*>(base + o_uinv);
    swapflags_ = reinterpret_cast<i32*>(base + o_flags);
    RL_CUDA_CHECK(cudaMemsetAsync(swapflags_, 0, sizeof(i32) * (leaf_of_.size() + 1), init_s));
    uready_ = reinterpret_cast<i32*>(base + o_uready);
    epoch_ = uready_ + leaf_of_.size() + 1;
    RL_CUDA_CHECK(cudaMemsetAsync(uready_, 0, sizeof(i32) * (leaf_of_.size() + 2), init_s));
    uflags_ = p_ <= 65536u && fused_trsm_ && RL_UREADY;
    leaf_starts_.assign(leaf_of_.size(), 0);
    for (const auto& kv : leaf_of_) leaf_starts_[kv.second] = kv.first;
    ninv_ = ninv_slot_.empty() ? nullptr : reinterpret_cast<u32*>(base + o_ninv);
    if (p_ <= 65536u) {
        inv_table_ = reinterpret_cast<uint16_t*>(base + o_tab);
        build_inv_table(inv_table_, p_, init_s);
    }
    RL_CUDA_CHECK(cudaStreamSynchronize(init_s));
    RL_CUDA_CHECK(cudaStreamDestroy(init_s));
    // the critical path (s_, s3_) outranks the wide updates (s2_) at the CTA
    // scheduler: a window CTA takes the first SM that frees up
    int prio_lo = 0, prio_hi = 0;
    RL_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    // s2_ (the rest of each Schur update, joined before the next tail) ranks
    // above the lanes when s2_prio_ (CTA dispatch order when SMs free up)
    RL_CUDA_CHECK(cudaStreamCreateWithPriority(&s2_, cudaStreamNonBlocking,
                                               s2_prio_ ? std::min(prio_lo, prio_hi + 1) : prio_lo));
    RL_CUDA_CHECK(cudaStreamCreateWithPriority(&s3_, cudaStreamNonBlocking, prio_hi));
    RL_CUDA_CHECK(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
    events_.resize(events_needed_ + 4);
    for (auto& e : events_) RL_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (a2_cap_) RL_CUDA_CHECK(cudaMalloc(&a2_, a2_cap_));
    if (b2_cap_) RL_CUDA_CHECK(cudaMalloc(&b2_, b2_cap_));
    for (auto& kv : lanes_) {
        Lane& l = kv.second;
        // a short lane's pieces are needed sooner: lanes of height 128, 256, ...
        // get the priorities right below the critical path's, the tall ones the lowest
        int prio = prio_lo;
        if (lane_prio_ && kv.first > 0) {
            int lvl = 0;
            for (i32 h = kv.first; h > 2 * PB; h /= 2) ++lvl;
            prio = std::min(prio_lo, prio_hi + 1 + lvl);
        }
        RL_CUDA_CHECK(cudaStreamCreateWithPriority(&l.st, cudaStreamNonBlocking, prio));
        if (l.a2_cap) RL_CUDA_CHECK(cudaMalloc(&l.a2, l.a2_cap));
        if (l.b2_cap) RL_CUDA_CHECK(cudaMalloc(&l.b2, l.b2_cap));
    }
    for (auto& kv : early_)
        if (kv.second.cap) RL_CUDA_CHECK(cudaMalloc(&kv.second.buf, kv.second.cap));
    if (!early_.empty()) RL_CUDA_CHECK(cudaStreamCreateWithPriority(&sb_, cudaStreamNonBlocking, prio_hi));
    if (!big_slot_.empty()) {
        RL_CUDA_CHECK(cudaMalloc(&big_, sizeof(u32) * BIG_LD * BIG_LD * big_slot_.size()));
        RL_CUDA_CHECK(cudaMalloc(&big_tmp_, sizeof(u32) * (4 * NINV_LD * NINV_LD + 4 * CH_LD * CH_LD)));
        RL_CUDA_CHECK(cudaStreamCreateWithPriority(&inv_lane_.st, cudaStreamNonBlocking, prio_lo));
        if (inv_lane_.a2_cap) RL_CUDA_CHECK(cudaMalloc(&inv_lane_.a2, inv_lane_.a2_cap));
        if (inv_lane_.b2_cap) RL_CUDA_CHECK(cudaMalloc(&inv_lane_.b2, inv_lane_.b2_cap));
    }
}

CupEngine::~CupEngine() {
    // an evicted engine may still have an asynchronous run in flight
    if (done_) cudaEventSynchronize(done_);
    if (done_) cudaEventDestroy(done_);
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    cudaFree(meta_);
    for (auto& e : events_) cudaEventDestroy(e);
    if (s2_) cudaStreamDestroy(s2_);
    if (s3_) cudaStreamDestroy(s3_);
    cudaFree(a2_);
    cudaFree(b2_);
    for (auto& kv : lanes_) {
        if (kv.second.st) cudaStreamDestroy(kv.second.st);
        cudaFree(kv.second.a2);
        cudaFree(kv.second.b2);
    }
    if (inv_lane_.st) cudaStreamDestroy(inv_lane_.st);
    cudaFree(inv_lane_.a2);
    cudaFree(inv_lane_.b2);
    cudaFree(big_);
    cudaFree(big_tmp_);
    for (auto& kv : early_) cudaFree(kv.second.buf);
    if (sb_) cudaStreamDestroy(sb_);
}

// Events shared with work outside the launch sequence (the host-buffer copy
// streams): external event nodes when the sequence is captured into a graph,
// plain records / waits when it is enqueued directly.
static bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    RL_CUDA_CHECK(cudaStreamIsCapturing(s, &st));
    return st == cudaStreamCaptureStatusActive;
}
void CupEngine::record_ext(cudaEvent_t e, cudaStream_t st) {
    if (capturing(st)) RL_CUDA_CHECK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else RL_CUDA_CHECK(cudaEventRecord(e, st));
}
void CupEngine::wait_ext(cudaStream_t st, cudaEvent_t e) {
    RL_CUDA_CHECK(cudaStreamWaitEvent(st, e, capturing(st) ? cudaEventWaitExternal : 0));
}

cudaEvent_t CupEngine::fork_to(cudaStream_t from, cudaStream_t to) {
    if (from == s_) flush_swaps();
    cudaEvent_t e = events_.at(next_event_++);
    RL_CUDA_CHECK(cudaEventRecord(e, from));
    RL_CUDA_CHECK(cudaStreamWaitEvent(to, e, 0));
    return e;
}

void CupEngine::gemm(i32 row0, i32 M, i32 x0, i32 x1, Dyn n_lo, Dyn n_hi, i64 Nmax, cudaStream_t st,
                     i32 n_cap, const EarlyPack* ep) {
    if (!st) st = work_stream();
    // K = pivots of rows [x0, x1) = [rp[x0], rp[x1]); split along the skeleton
    // while the s32 exactness bound could be exceeded.
    const i64 Kmax = x1 - x0;
    if (Kmax <= 0 || M <= 0 || Nmax <= 0) return;
    if (Kmax > tc_kmax(L_)) {
        if (ep) throw Error(7 /*RL_EINVAL*/, "early B pack of a K-split GEMM");
        const i32 xm = x0 + (x1 - x0) / 2;
        gemm(row0, M, x0, xm, n_lo, n_hi, Nmax, st, n_cap);
        gemm(row0, M, xm, x1, n_lo, n_hi, Nmax, st, n_cap);
        return;
    }
    // side-lane work packs into its lane's own workspace
    Lane* ln = (lane_ && st == lane_->st) ? lane_ : nullptr;
    GemmArgs g{};
    g.A = A_;
    g.lda = lda_;
    g.a_row0 = row0;
    g.B = A_;
    g.ldb = lda_;
    g.gather = rrp_;
    g.C = A_;
    g.ldc = lda_;
    g.c_row0 = row0;
    g.M = M;
    g.k_lo = dyn_rp(x0);
    g.k_hi = dyn_rp(x1);
    g.n_lo = n_lo;
    g.n_hi = n_hi;
    g.rp = rp_;
    g.n_cap = n_cap;
    // on the side stream the persistent GEMM leaves one SM for the window kernel
#ifndef RL_SIDE_FREE_SMS
#define RL_SIDE_FREE_SMS 1
#endif
    g.max_ctas = (st == s_)                           ? 0
                 : (ln && is_tile_lane(ln))            ? tile_ctas_
                 : (ln && lane_ctas_ > 0)              ? lane_ctas_
                                                       : num_sms() - RL_SIDE_FREE_SMS;
    g.alpha = p_ - 1;  // C <- C - A*B  (mm(..., neg_one, one), factor.cpp:51)
    g.beta = 1 % p_;
    g.f = f_;
    // skinny K (one leaf): the SIMT kernel reads the operands directly and
    // beats packing them for the tensor cores
    // ... and so are the 128-column window slices of the split updates up to K = 256
#ifndef RL_IMMA_MAX_K
#define RL_IMMA_MAX_K PB
#endif
#ifndef RL_IMMA_MAX_MK
#define RL_IMMA_MAX_MK 0
#endif
    // (p <= 2^16: small updates, K <= RL_IMMA_MAX_K or M*K <= RL_IMMA_MAX_MK, skip the packing too)
    const bool small = p_ <= 65536u && (Kmax <= RL_IMMA_MAX_K || (i64)M * Kmax <= (i64)RL_IMMA_MAX_MK);
    const bool tc = use_tc_ && !small && Kmax > PB && Nmax >= 64 && M >= 64 && !(Nmax <= PW && Kmax <= 4 * PB);
    if (dry_) {
        if (tc) {
            size_t& ac = ln ? ln->a2_cap : a2_cap_;
            size_t& bc = ln ? ln->b2_cap : b2_cap_;
            ac = std::max(ac, tc_a2_bytes(L_, M, Kmax));
            bc = std::max(bc, tc_b2_bytes(L_, Nmax, Kmax));
        }
        return;
    }
    if (st == s_) flush_swaps();
    ++stats_.gemms;
    if (tc && ep && ep->buf) {  // B packed earlier on sb_
        ++stats_.tc_gemms;
        stats_.launches += 2;
        RL_CUDA_CHECK(cudaStreamWaitEvent(st, ep->ev, 0));
        gemm_tc_split(g, L_, Kmax, Nmax, ln ? ln->a2 : a2_, ep->buf, st, 3);
    } else if (tc) {
        ++stats_.tc_gemms;
        stats_.launches += 2;
        gemm_tc(g, L_, Kmax, Nmax, ln ? ln->a2 : a2_, ln ? ln->b2 : b2_, st);
    } else {
        stats_.launches += 1;
        gemm_simt(g, Kmax, Nmax, st);
    }
}

void CupEngine::panel(i32 i0, i32 b) {
    if (dry_) {
        leaf_of_.emplace(i0, (i32)leaf_of_.size());
        events_needed_ += 2;
        return;
    }
    flush_swaps();
    PanelArgs a{};
    a.uinv = uinv_ + (size_t)leaf_of_.at(i0) * PB * PB;
    a.swapflag = swapflags_ + leaf_of_.at(i0);
    a.uready = uready_ + leaf_of_.at(i0);
    a.epoch = epoch_;
    a.inv_table = inv_table_;
    a.A = A_;
    a.lda = lda_;
    a.i0 = i0;
    a.b = b;
    a.N = n_;
    a.rp = rp_;
    a.rrp = rrp_;
    a.ipiv = ipiv_;
    a.ps = ps_;
    a.f = f_;
    panel_window(a, s_);
    if (!RL_UINV_IN_TAIL) {
        fork_to(s_, s3_);                   // U^{-1} beside the tail
        panel_uinv(a, s3_);
    }
    // a joined side-stream kernel may become a programmatic predecessor of the
    // tail and still be writing these rows when its CTAs start: no prefetch then
    a.prefetch = pending_joins_.empty() ? 1 : 0;
    for (cudaEvent_t e : pending_joins_) RL_CUDA_CHECK(cudaStreamWaitEvent(s_, e, 0));
    pending_joins_.clear();                 // the wide Schur update of these rows
    panel_tail(a, s_);
    // U^{-1} (and the panel scratch it reads) is joined before the next TRSM,
    // which always precedes the next window: the swaps in between overlap it
    if (!RL_UINV_IN_TAIL) {
        uinv_join_ = events_.at(next_event_++);
        RL_CUDA_CHECK(cudaEventRecord(uinv_join_, s3_));
    } else {
        ++next_event_;  // (keeps the dry run's event count valid)
    }
    stats_.panels++;
    stats_.launches += 3;
}

void CupEngine::leaf_range(i32 piv_lo, i32 piv_hi, SwapArgs& a) const {
    a.leafflags = swapflags_;
    a.leaf_lo = (i32)(std::lower_bound(leaf_starts_.begin(), leaf_starts_.end(), piv_lo) - leaf_starts_.begin());
    a.leaf_hi = (i32)(std::lower_bound(leaf_starts_.begin(), leaf_starts_.end(), piv_hi) - leaf_starts_.begin());
}

void CupEngine::swaps_range(i32 row0, i32 M, Dyn j_lo, Dyn j_hi, i32 piv_lo, i32 piv_hi) {
    if (dry_ || M <= 0) return;
    SwapArgs a{};
    a.A = A_;
    a.lda = lda_;
    a.row0 = row0;
    a.M = M;
    a.gather = nullptr;
    a.j_lo = j_lo;
    a.j_hi = j_hi;
    a.rp = rp_;
    a.ipiv = ipiv_;
    a.Mmax = M;
    leaf_range(piv_lo, piv_hi, a);
    queue_swaps(a);
}

// swaps_range as its own launch on stream st (side-lane work)
void CupEngine::swaps_range_on(cudaStream_t st, i32 row0, i32 M, Dyn j_lo, Dyn j_hi, i32 piv_lo, i32 piv_hi) {
    if (dry_ || M <= 0) return;
    SwapJobs jobs{};
    SwapArgs& a = jobs.job[0];
    a.A = A_;
    a.lda = lda_;
    a.row0 = row0;
    a.M = M;
    a.gather = nullptr;
    a.j_lo = j_lo;
    a.j_hi = j_hi;
    a.rp = rp_;
    a.ipiv = ipiv_;
    a.Mmax = M;
    leaf_range(piv_lo, piv_hi, a);
    jobs.n = 1;
    apply_swaps(jobs, st);
    stats_.launches += 1;
}

void CupEngine::swaps_gather(Dyn g_lo, Dyn g_hi, i32 Mmax, Dyn j_lo, Dyn j_hi, i32 piv_lo, i32 piv_hi) {
    if (dry_ || Mmax <= 0) return;
    SwapArgs a{};
    a.A = A_;
    a.lda = lda_;
    a.gather = rrp_;
    a.g_lo = g_lo;
    a.g_hi = g_hi;
    a.j_lo = j_lo;
    a.j_hi = j_hi;
    a.rp = rp_;
    a.ipiv = ipiv_;
    a.Mmax = Mmax;
    leaf_range(piv_lo, piv_hi, a);
    queue_swaps(a);
}

// Swap jobs are queued and launched together right before the next kernel on
// the critical path (consecutive jobs touch disjoint rows, see perm.cu).
void CupEngine::queue_swaps(const SwapArgs& a) {
    if (swap_jobs_.n == MAX_SWAP_JOBS) flush_swaps();
    swap_jobs_.job[swap_jobs_.n++] = a;
}

void CupEngine::flush_swaps() {
    if (dry_ || swap_jobs_.n == 0) return;
    apply_swaps(swap_jobs_, s_);
    swap_jobs_.n = 0;
    stats_.launches += 1;
}

// G <- G * U_X^{-1} for the unit upper block of node X = rows [x0, x0+mx)
// (trsm Right/Upper/Unit, kernels.cpp:149-154, recursing along X's own skeleton).
static void collect_leaves(i32 x0, i32 mx, std::vector<std::pair<i32, i32>>& out) {
    if (mx <= PB) {
        out.emplace_back(x0, mx);
        return;
    }
    collect_leaves(x0, mx / 2, out);
    collect_leaves(x0 + mx / 2, mx - mx / 2, out);
}

// G <- G * U_X^{-1} as one GEMM against the stored node inverse (in place: the
// pack kernel snapshots G before the GEMM overwrites it, beta = 0).
void CupEngine::gemm_ninv(i32 r0, i32 M, i32 x0, i32 mx, const u32* ninv, i32 ldn) {
    GemmArgs g{};
    g.A = A_;
    g.lda = lda_;
    g.a_row0 = r0;
    g.B = ninv;
    g.ldb = ldn;
    g.gather = nullptr;
    g.b_from0 = 1;
    g.C = A_;
    g.ldc = lda_;
    g.c_row0 = r0;
    g.M = M;
    g.k_lo = dyn_rp(x0);
    g.k_hi = dyn_rp(x0 + mx);
    g.n_lo = dyn_rp(x0);
    g.n_hi = dyn_rp(x0 + mx);
    g.rp = rp_;
    g.alpha = 1 % p_;
    g.beta = 0;
    g.f = f_;
    flush_swaps();
    ++stats_.gemms;
    ++stats_.tc_gemms;
    stats_.launches += 2;
    if (lane_) g.max_ctas = is_tile_lane(lane_) ? tile_ctas_ : lane_ctas_ > 0 ? lane_ctas_ : num_sms() - 1;
    gemm_tc(g, L_, mx, mx, lane_ ? lane_->a2 : a2_, lane_ ? lane_->b2 : b2_, work_stream());
}

void CupEngine::trsm_right(i32 r0, i32 M, i32 x0, i32 mx) {
    // a tall TRSM against a node with a big inverse: one GEMM (the inverse is
    // unique, so the bytes are the reference recursion's)
    // (not the node factored last before this TRSM: its inverse is still being
    // built, the recursion below is faster than waiting for it)
    if (big_on_ && use_tc_ && (M >= kBigMinRows || is_tile_lane(lane_)) && x0 + mx < trsm_end_) {
        const auto key = std::make_pair(x0, mx);
        if (big_slot_.count(key)) {
            if (dry_) {
                size_t& ac = lane_ ? lane_->a2_cap : a2_cap_;
                size_t& bc = lane_ ? lane_->b2_cap : b2_cap_;
                ac = std::max(ac, tc_a2_bytes(L_, M, mx));
                bc = std::max(bc, tc_b2_bytes(L_, mx, mx));
                return;
            }
            auto it = big_ready_.find(key);
            if (it != big_ready_.end()) {
                flush_swaps();
                RL_CUDA_CHECK(cudaStreamWaitEvent(work_stream(), it->second, 0));
                gemm_ninv(r0, M, x0, mx, big_ + (size_t)big_slot_.at(key) * BIG_LD * BIG_LD, BIG_LD);
                return;
            }
        }
    }
    if (fused_trsm_ && mx <= TN_MAXLEAF * PB) {  // <= 4 leaves: one fused kernel
        const auto key = std::make_pair(x0, mx);
        const bool gemm_ok = use_tc_ && M >= kNinvGemmMinRows && mx >= 2 * PB;
        if (dry_) {
            if (!ninv_slot_.count(key)) ninv_slot_.emplace(key, (i32)ninv_slot_.size());
            if (gemm_ok) {
                size_t& ac = lane_ ? lane_->a2_cap : a2_cap_;
                size_t& bc = lane_ ? lane_->b2_cap : b2_cap_;
                ac = std::max(ac, tc_a2_bytes(L_, M, mx));
                bc = std::max(bc, tc_b2_bytes(L_, mx, mx));
            }
            return;
        }
        u32* ninv = ninv_ + (size_t)ninv_slot_.at(key) * NINV_LD * NINV_LD;
        const bool have = ninv_done_.count(key) != 0;
        if (have && gemm_ok) {
            gemm_ninv(r0, M, x0, mx, ninv);
            return;
        }
        std::vector<std::pair<i32, i32>> lv;
        collect_leaves(x0, mx, lv);
        TrsmNodeArgs a{};
        a.A = A_;
        a.lda = lda_;
        a.row0 = r0;
        a.M = M;
        a.nleaf = (int)lv.size();
        for (int l = 0; l < a.nleaf; ++l) {
            a.j_lo[l] = dyn_rp(lv[l].first);
            a.j_hi[l] = dyn_rp(lv[l].first + lv[l].second);
            a.uinv[l] = uinv_ + (size_t)leaf_of_.at(lv[l].first) * PB * PB;
            a.uready[l] = uflags_ ? uready_ + leaf_of_.at(lv[l].first) : nullptr;
        }
        a.epoch = epoch_;
        a.rp = rp_;
        a.rrp = rrp_;
        a.f = f_;
        flush_swaps();
        // first TRSM against X also leaves U_X^{-1} -- only where a taller TRSM can
        // use it: a node of more than two leaves (a TRSM against a node of <= 2
        // leaves solves at most as many rows as the node has, M < kNinvGemmMinRows)
        const bool want = !have && mx > 2 * PB;
        a.ninv = want ? ninv : nullptr;
        if (want) ninv_done_.insert(key);
        trsm_node(a, work_stream());
        stats_.trsm_leaves++;
        stats_.launches += 1;
        return;
    }
    if (mx <= PB) {
        if (dry_) return;
        TrsmLeafArgs a{};
        a.A = A_;
        a.lda = lda_;
        a.row0 = r0;
        a.M = M;
        a.j_lo = dyn_rp(x0);
        a.j_hi = dyn_rp(x0 + mx);
        a.rp = rp_;
        a.uinv = uinv_ + (size_t)leaf_of_.at(x0) * PB * PB;
        a.f = f_;
        flush_swaps();
        trsm_leaf(a, work_stream());
        stats_.trsm_leaves++;
        stats_.launches += 1;
        return;
    }
    const i32 kx = mx / 2;
    trsm_right(r0, M, x0, kx);
    gemm(r0, M, x0, x0 + kx, dyn_rp(x0 + kx), dyn_rp(x0 + mx), mx - kx);
    trsm_right(r0, M, x0 + kx, mx - kx);
}

// The bridge of the leaf of rows [leaf, leaf_end) (its pivots, U^{-1},
// transposition flag) into rows [row0, row0 + M), slice from n_lo (bridge.cu).
BridgeArgs CupEngine::leaf_bridge(i32 leaf, i32 leaf_end, i32 row0, i32 M, Dyn n_lo) const {
    BridgeArgs a{};
    a.A = A_;
    a.lda = lda_;
    a.row0 = row0;
    a.M = M;
    a.j_lo = dyn_rp(leaf);
    a.j_hi = dyn_rp(leaf_end);
    a.n_lo = n_lo;
    a.N = n_;
    a.rp = rp_;
    a.rrp = rrp_;
    a.ipiv = ipiv_;
    a.uinv = uinv_ + (size_t)leaf_of_.at(leaf) * PB * PB;
    a.uready = uflags_ ? uready_ + leaf_of_.at(leaf) : nullptr;
    a.epoch = epoch_;
    a.swapflag = swapflags_ + leaf_of_.at(leaf);
    a.ps = ps_;
    a.f = f_;
    return a;
}

// The limb image of the Schur update's B operand (the U rows of node (i0, mm)'s
// top half [i0, i0 + k), gathered through rrp, at columns [rp[i0 + k], n)) on
// sb_, right after the top half is factored: the GEMMs that read it (the
// critical one and the row-split lane's) then pack only their A operand.
// Same GemmArgs fields as gemm() builds for them, so the same image.
CupEngine::EarlyPack CupEngine::early_pack_b(i32 i0, i32 k, i32 mm) {
    EarlyPack ep{};
    const i32 b0 = i0 + k;
    EarlyBuf& eb = early_[mm];
    if (dry_) {
        eb.cap = std::max(eb.cap, tc_b2_bytes(L_, n_, k));
        events_needed_ += 2;
        return ep;
    }
    GemmArgs g{};
    g.A = A_;
    g.lda = lda_;
    g.B = A_;
    g.ldb = lda_;
    g.gather = rrp_;
    g.C = A_;
    g.ldc = lda_;
    g.M = 1;
    g.k_lo = dyn_rp(i0);
    g.k_hi = dyn_rp(b0);
    g.n_lo = dyn_rp(b0);
    g.n_hi = dyn_c(n_);
    g.rp = rp_;
    g.f = f_;
    fork_to(s_, sb_);  // the top half's U rows are final (its swaps flushed)
    gemm_tc_split(g, L_, k, n_, nullptr, eb.buf, sb_, 4);
    stats_.launches += 1;
    ep.buf = eb.buf;
    ep.ev = events_.at(next_event_++);
    RL_CUDA_CHECK(cudaEventRecord(ep.ev, sb_));
    early_used_ = true;
    return ep;
}

void CupEngine::node(i32 i0, i32 mm) {
    if (mm <= PB) {
        panel(i0, mm);
        return;
    }
    const i32 k = mm / 2;                    // factor.cpp:35
    node(i0, k);                             // factor.cpp:39
    if (!dry_ && !dones_.empty() && !tiling_) {  // this node's top half is factored
        auto it = dones_.find({i0, mm});
        if (it != dones_.end()) {
            flush_swaps();
            record_ext(it->second, s_);
        }
    }
    if (!dry_ && !waits_.empty()) {  // its bottom rows may still be arriving from the host
        auto it = waits_.find({i0, mm});
        if (it != waits_.end()) wait_ext(s_, it->second);
    }
    if (!dry_) {  // the lower rows' TRSM + Schur update ran on a side lane
        auto it = row_joins_.find({i0, mm});
        if (it != row_joins_.end()) {
            RL_CUDA_CHECK(cudaStreamWaitEvent(s_, it->second, 0));
            row_joins_.erase(it);
        }
    }
    const i32 b0 = i0 + k, bm = mm - k;
    trsm_end_ = b0;  // the TRSMs of this node solve against rows [i0, b0)
    // the wide Schur update (k > split_max_k_, tensor cores, one K chunk): its
    // B operand is packed now, beside the TRSM
    EarlyPack ep{};
    const bool early = early_b_on_ && use_tc_ && !geo_split_ && k > split_max_k_ && k > PB &&
                       k <= tc_kmax(L_) && bm >= 64 && n_ - k >= 64;
    if (early) ep = early_pack_b(i0, k, mm);
    // (dry run: ep.buf is null but the GEMM sizing must see the early pack too;
    // a K-split GEMM never gets one)
    const EarlyPack* epp = early && (ep.buf || dry_) ? &ep : nullptr;
    // a leaf pair (top = one leaf, p <= 2^16): swaps, TRSM and the window slice's
    // update in one launch (bridge.cu)
    const bool br = bridge_on_ && k <= PB && bm <= PB && p_ <= 65536u && use_tc_;
    if (!br) {
        swaps_range(b0, bm, dyn_rp(i0), dyn_rp(b0), i0, b0);   // factor.cpp:42
        // launched now, so it runs beside the last leaf's U^{-1} (joined below)
        // instead of after it on the critical path
        flush_swaps();
    }
    if (!dry_ && uinv_join_ && !uflags_) {  // (with the flags its readers wait on the device)
        RL_CUDA_CHECK(cudaStreamWaitEvent(s_, uinv_join_, 0));
        uinv_join_ = nullptr;
    }
    // factor.cpp:51-52, split: the first window of the bottom half reads only
    // columns [rp[b0], rp[b0] + PW), so that slice is updated first and the rest
    // runs on s2_ beside that window (joined before its tail)
    if (geo_split_ && bm > PB && k <= geo_max_k_) {
        // Geometric row split.  The bottom recursion node(b0, bm) first touches
        // its rows in the order of its left spine: the leaf [b0, b0 + s_L), then
        // the bottom half [b0 + s/2, b0 + s) of node(b0, s) for s = 2 s_L, ..., bm
        // (each right after node(b0, s)'s top half is factored).  Only the first
        // leaf's TRSM + window-slice update runs on the critical path; every
        // later piece's TRSM + full-width Schur update runs, smallest (= needed
        // soonest) first, on the low-priority lane of height bm and is joined by
        // node(b0, s) right before its first touch of those rows (row_joins_).
        // Value-neutral: row blocks of a right TRSM and of a Schur update are
        // independent, and no piece row is read or written by anything else
        // before its join.
        std::vector<i32> spine;  // s = bm, bm/2, ... (> PB): node(b0, s) on the left spine
        for (i32 s = bm; s > PB; s /= 2) spine.push_back(s);
        const i32 leaf = spine.back() / 2;  // node(b0, leaf) is the first leaf
        trsm_right(b0, leaf, i0, k);                                   // factor.cpp:45-46
        gemm(b0, leaf, i0, b0, dyn_rp(b0), Dyn{b0, PW}, std::min<i64>(PW, n_), s_, n_);
        if (dry_) {
            events_needed_ += 2;
            gemm(b0, leaf, i0, b0, Dyn{b0, PW}, dyn_c(n_), n_, s2_);
        } else {
            fork_to(s_, s2_);
            gemm(b0, leaf, i0, b0, Dyn{b0, PW}, dyn_c(n_), n_, s2_);
            cudaEvent_t e = events_.at(next_event_++);
            RL_CUDA_CHECK(cudaEventRecord(e, s2_));
            pending_joins_.push_back(e);
        }
        Lane& ln = lanes_[bm];
        if (dry_) events_needed_ += 1 + spine.size();
        else fork_to(s_, ln.st);
        lane_ = &ln;
        for (size_t q = spine.size(); q-- > 0;) {
            const i32 s = spine[q], h = s / 2;
            trsm_right(b0 + h, s - h, i0, k);
            gemm(b0 + h, s - h, i0, b0, dyn_rp(b0), dyn_c(n_), n_);
            if (!dry_) {
                cudaEvent_t e = events_.at(next_event_++);
                RL_CUDA_CHECK(cudaEventRecord(e, ln.st));
                row_joins_[{b0, s}] = e;
            }
        }
        lane_ = nullptr;
    } else if (k > split_max_k_ && row_split_min_ > 0 && bm >= row_split_min_ && bm > 2 * PB) {
        // rows [b0, b0 + h) now; rows [b0 + h, b0 + bm) on the lane of height bm,
        // joined in node(b0, bm) after its top half (rows [b0, b0 + h)) is factored
        const i32 h = bm / 2;
        trsm_right(b0, h, i0, k);                                     // factor.cpp:45-46
        gemm(b0, h, i0, b0, dyn_rp(b0), dyn_c(n_), n_, nullptr, 0, epp);
        Lane& ln = lanes_[bm];
        if (dry_) {
            events_needed_ += 2;
        } else {
            fork_to(s_, ln.st);
        }
        lane_ = &ln;
        trsm_right(b0 + h, bm - h, i0, k);
        gemm(b0 + h, bm - h, i0, b0, dyn_rp(b0), dyn_c(n_), n_, nullptr, 0, epp);
        lane_ = nullptr;
        if (!dry_) {
            cudaEvent_t e = events_.at(next_event_++);
            RL_CUDA_CHECK(cudaEventRecord(e, ln.st));
            row_joins_[{b0, bm}] = e;
        }
    } else if (br) {
        if (!dry_) {
            BridgeArgs a = leaf_bridge(i0, b0, b0, bm, dyn_rp(b0));
            flush_swaps();
            bridge(a, s_);
            stats_.launches += 1;
        }
        if (dry_) {
            events_needed_ += 2;
            gemm(b0, bm, i0, b0, Dyn{b0, PW}, dyn_c(n_), n_, s2_);
        } else {
            fork_to(s_, s2_);
            gemm(b0, bm, i0, b0, Dyn{b0, PW}, dyn_c(n_), n_, s2_);
            cudaEvent_t e = events_.at(next_event_++);
            RL_CUDA_CHECK(cudaEventRecord(e, s2_));
            pending_joins_.push_back(e);
        }
    } else if (k > split_max_k_) {
        trsm_right(b0, bm, i0, k);                                    // factor.cpp:45-46
        gemm(b0, bm, i0, b0, dyn_rp(b0), dyn_c(n_), n_, nullptr, 0, epp);
    } else {
        trsm_right(b0, bm, i0, k);                                    // factor.cpp:45-46
        gemm(b0, bm, i0, b0, dyn_rp(b0), Dyn{b0, PW}, std::min<i64>(PW, n_), s_, n_);
        rest_update(b0, bm, i0, b0);
    }
    node(b0, bm);                                                     // factor.cpp:53
    swaps_gather(dyn_rp(i0), dyn_rp(b0), k, dyn_rp(b0), dyn_rp(i0 + mm), b0, i0 + mm);  // factor.cpp:56
    if (big_on_ && use_tc_ && mm > 8 * PB && mm <= BIG_LD && m_ >= 2 * kBigMinRows) build_big_inverse(i0, mm);
}

// The Schur update of rows [b0, b0 + bm) against the pivots of rows [x0, x1)
// beyond the slice the next window reads (columns >= rp[b0] + PW), on s2_
// beside that window.  In pieces along node(b0, bm)'s left spine when
// rest_pieces_: the first leaf's rows first (joined before its tail), then
// the bottom half of node(b0, s) for s = 2 x leaf, ..., bm (joined by node(b0, s)
// right before its first touch of those rows, see node()), so a leaf's tail
// never waits for rows it does not read -- the pieces needed first are the
// smallest and are done first even when a side lane holds most SMs.
// Returns the event of the last piece.
cudaEvent_t CupEngine::rest_update(i32 b0, i32 bm, i32 x0, i32 x1) {
    std::vector<i32> spine;  // s_0 = bm, s_{t+1} = s_t / 2 (node()'s split) down to the first leaf
    if (rest_pieces_) {
        for (i32 s = bm;; s /= 2) {
            spine.push_back(s);
            if (s <= PB) break;
        }
    } else {
        spine.push_back(bm);
    }
    if (dry_) events_needed_ += 2 + spine.size();
    else fork_to(s_, s2_);
    cudaEvent_t e = nullptr;
    auto record = [&](cudaStream_t st) {
        if (dry_) return (cudaEvent_t) nullptr;
        cudaEvent_t ev = events_.at(next_event_++);
        RL_CUDA_CHECK(cudaEventRecord(ev, st));
        return ev;
    };
    // rest_split_ (one tensor-core K chunk): the rows of the first leaf pair first
    // -- the first tail waits for that GEMM only -- then the rows below with the B
    // image the first GEMM packed (same stream, same workspace), joined by the
    // left-spine node whose bottom half starts there, right before its first
    // touch of those rows
    if (rest_split_ && !rest_pieces_ && use_tc_ && x1 - x0 > PB && x1 - x0 <= tc_kmax(L_) && n_ > 2 * PW) {
        i32 hi = bm, lo = bm / 2;  // node(b0, hi) has its bottom half at b0 + lo
        while (lo / 2 >= 2 * PB) {
            hi = lo;
            lo /= 2;
        }
        if (lo >= 2 * PB && lo < bm && (dry_ || row_joins_.find({b0, hi}) == row_joins_.end())) {
            if (dry_) events_needed_ += 4;
            gemm(b0, lo, x0, x1, Dyn{b0, PW}, dyn_c(n_), n_, s2_);
            e = record(s2_);
            if (!dry_) pending_joins_.push_back(e);
            if (rest_split_ == 2) {
                // ... on the lane of this height (own stream and workspaces, its own B
                // pack): the later, smaller rest updates on s2_ do not queue behind it
                Lane& ln = lanes_[bm];
                if (!dry_) fork_to(s_, ln.st);
                Lane* saved = lane_;
                lane_ = &ln;
                gemm(b0 + lo, bm - lo, x0, x1, Dyn{b0, PW}, dyn_c(n_), n_);
                e = record(ln.st);
                lane_ = saved;
            } else {
                EarlyPack ep{};
                ep.buf = b2_;
                ep.ev = e;
                gemm(b0 + lo, bm - lo, x0, x1, Dyn{b0, PW}, dyn_c(n_), n_, s2_, 0, &ep);
                e = record(s2_);
            }
            if (!dry_) row_joins_[{b0, hi}] = e;
            return e;
        }
    }
    const i32 l0 = spine.back();
    gemm(b0, l0, x0, x1, Dyn{b0, PW}, dyn_c(n_), n_, s2_);
    e = record(s2_);
    if (!dry_) pending_joins_.push_back(e);
    if (spine.size() > 1) {
        // the later pieces on the lane of this height (own stream and GEMM
        // workspace): they are joined deep in the recursion, while s_ and s2_
        // keep packing into their own workspaces
        Lane& ln = lanes_[bm];
        if (!dry_) fork_to(s_, ln.st);
        Lane* saved = lane_;
        lane_ = &ln;
        for (int t = (int)spine.size() - 2; t >= 0; --t) {
            const i32 lo = spine[t + 1], hi = spine[t];
            gemm(b0 + lo, hi - lo, x0, x1, Dyn{b0, PW}, dyn_c(n_), n_);
            e = record(ln.st);
            if (!dry_) row_joins_[{b0, hi}] = e;
        }
        lane_ = saved;
    }
    return e;
}

// C <- alpha * A * B (beta = 0) on dense / gathered operands, on stream st
// with the inverse lane's workspace.
void CupEngine::gemm_dense(const u32* A, i64 lda, bool a_dense, const u32* B, i64 ldb, bool b_dense,
                           const i32* gather, u32* C, i64 ldc, i32 M, Dyn k_lo, Dyn k_hi, Dyn n_lo, Dyn n_hi,
                           i64 Kmax, i64 Nmax, u32 alpha, cudaStream_t st) {
    if (dry_) {
        inv_lane_.a2_cap = std::max(inv_lane_.a2_cap, tc_a2_bytes(L_, M, Kmax));
        inv_lane_.b2_cap = std::max(inv_lane_.b2_cap, tc_b2_bytes(L_, Nmax, Kmax));
        return;
    }
    GemmArgs g{};
    g.A = A;
    g.lda = lda;
    g.a_from0 = a_dense ? 1 : 0;
    g.B = B;
    g.ldb = ldb;
    g.b_from0 = b_dense ? 1 : 0;
    g.gather = gather;
    g.C = C;
    g.ldc = ldc;
    g.c_from0 = 1;
    g.M = M;
    g.k_lo = k_lo;
    g.k_hi = k_hi;
    g.n_lo = n_lo;
    g.n_hi = n_hi;
    g.rp = rp_;
    g.alpha = alpha;
    g.beta = 0;
    g.f = f_;
    ++stats_.gemms;
    ++stats_.tc_gemms;
    stats_.launches += 2;
    gemm_tc(g, L_, Kmax, Nmax, inv_lane_.a2, inv_lane_.b2, st);
}

// X = U^{-1} of the node [a | b] from Xa, Xb:  X = [[Xa, -Xa U_ab Xb], [0, Xb]],
// U_ab = the U rows of a's pivots (gathered through rrp) at b's pivot columns.
void CupEngine::combine_inverse(const u32* Xa, i32 la, i32 xa, i32 ma, const u32* Xb, i32 lb, i32 xb, i32 mb,
                                u32* X, i32 ldx, cudaStream_t st) {
    u32* T1 = big_tmp_ ? big_tmp_ + 4 * NINV_LD * NINV_LD + 2 * CH_LD * CH_LD : nullptr;
    u32* T2 = T1 ? T1 + CH_LD * CH_LD : nullptr;
    gemm_dense(Xa, la, true, A_, lda_, false, rrp_, T1, CH_LD, ma, dyn_rp(xa), dyn_rp(xb), dyn_rp(xb),
               dyn_rp(xb + mb), ma, mb, 1 % p_, st);
    gemm_dense(T1, CH_LD, true, Xb, lb, true, nullptr, T2, CH_LD, ma, dyn_rp(xb), dyn_rp(xb + mb), dyn_rp(xb),
               dyn_rp(xb + mb), mb, mb, p_ - 1, st);
    if (!dry_) {
        ninv_assemble(X, ldx, Xa, la, Xb, lb, T2, CH_LD, dyn_rp(xa), dyn_rp(xb), dyn_rp(xb + mb), rp_, ma + mb, st);
        stats_.launches += 1;
    }
}

void CupEngine::build_big_inverse(i32 x0, i32 mm) {
    const auto key = std::make_pair(x0, mm);
    if (dry_) {
        if (!big_slot_.count(key)) big_slot_.emplace(key, (i32)big_slot_.size());
        events_needed_ += 2;
    } else {
        fork_to(s_, inv_lane_.st);  // the node's U rows are final (its swaps flushed)
        // ... and its last leaf's U^{-1} (still on s3_; s_ joins it later)
        if (uinv_join_) RL_CUDA_CHECK(cudaStreamWaitEvent(inv_lane_.st, uinv_join_, 0));
    }
    cudaStream_t st = inv_lane_.st;
    const i32 k = mm / 2;
    const i32 cx[2] = {x0, x0 + k}, cm[2] = {k, mm - k};
    u32* child[2] = {nullptr, nullptr};
    for (int c = 0; c < 2; ++c) {
        // the child's two halves (<= 4 leaves each): inverses by the fused
        // node solve with no rows (a private copy: the critical path may be
        // writing the shared slot of the same node at the same time)
        const i32 h = cm[c] / 2;
        const i32 gx[2] = {cx[c], cx[c] + h}, gm[2] = {h, cm[c] - h};
        u32* gi[2];
        for (int q = 0; q < 2; ++q) {
            gi[q] = big_tmp_ ? big_tmp_ + (size_t)(2 * c + q) * NINV_LD * NINV_LD : nullptr;
            if (dry_) continue;
            std::vector<std::pair<i32, i32>> lv;
            collect_leaves(gx[q], gm[q], lv);
            TrsmNodeArgs a{};
            a.A = A_;
            a.lda = lda_;
            a.row0 = 0;
            a.M = 0;
            a.nleaf = (int)lv.size();
            for (int l = 0; l < a.nleaf; ++l) {
                a.j_lo[l] = dyn_rp(lv[l].first);
                a.j_hi[l] = dyn_rp(lv[l].first + lv[l].second);
                a.uinv[l] = uinv_ + (size_t)leaf_of_.at(lv[l].first) * PB * PB;
                a.uready[l] = uflags_ ? uready_ + leaf_of_.at(lv[l].first) : nullptr;
            }
            a.epoch = epoch_;
            a.rp = rp_;
            a.rrp = rrp_;
            a.f = f_;
            a.ninv = gi[q];
            trsm_node(a, st);
            stats_.launches += 1;
        }
        child[c] = big_tmp_ ? big_tmp_ + 4 * NINV_LD * NINV_LD + (size_t)c * CH_LD * CH_LD : nullptr;
        combine_inverse(gi[0], NINV_LD, gx[0], gm[0], gi[1], NINV_LD, gx[1], gm[1], child[c], CH_LD, st);
    }
    u32* X = (big_ && !dry_) ? big_ + (size_t)big_slot_.at(key) * BIG_LD * BIG_LD : nullptr;
    combine_inverse(child[0], CH_LD, cx[0], cm[0], child[1], CH_LD, cx[1], cm[1], X, BIG_LD, st);
    if (!dry_) {
        cudaEvent_t e = events_.at(next_event_++);
        RL_CUDA_CHECK(cudaEventRecord(e, st));
        big_ready_[key] = e;
    }
}

// Tiled top level.  The reference's recursion (factor.cpp:35-53) updates the
// bottom half of a node only after its whole top half is factored, so at the
// upper levels the next leaf waits for a tall TRSM (a chain of dependent
// GEMMs along the top half's skeleton) and a wide Schur GEMM.  Here the rows
// are cut into tiles P_0, P_1, ... of g rows; P_j is factored by node() (the
// recursion, unchanged), then every row below receives P_j's transpositions,
// its TRSM against U_Pj and its Schur update (right-looking at the tile
// level).  Only the NEXT tile's rows are updated on the critical path; the
// rows below it are updated on a side lane beside the next tile's recursion
// (which leaves most SMs idle: its leaf chain is latency-bound).  The
// elimination is the same, grouped differently: with the reference's pivot
// rule the packed [C\U], the row profile and sigma are unique (SURVEY.md 8(c),
// "iterative formulation"), so the bytes are the recursion's.  The OpCounter
// is computed from the reference skeleton (cup_opcount), not from this order.
void CupEngine::tiled(i32 g) {
    tiling_ = true;  // node() leaves the host-overlap "done" records to this loop
    const i32 ntiles = (m_ + g - 1) / g;
    // Rows still arriving from the host (host-buffer path): pieces [lo, hi) with
    // the event of their copy; rows below the first piece are resident at launch.
    // Either per tile (set_host_rows) or the left-spine halves (set_host_overlap).
    std::vector<std::pair<std::pair<i32, i32>, cudaEvent_t>> arrive = host_in_;
    if (arrive.empty())
        for (const auto& kv : waits_)
            if (kv.first.first == 0) arrive.push_back({{kv.first.second / 2, kv.first.second}, kv.second});
    std::sort(arrive.begin(), arrive.end(),
              [](const auto& x, const auto& y) { return x.first.first < y.first.first; });
    auto wait_rows = [&](cudaStream_t st, i32 lo, i32 hi) {
        if (dry_) return;
        for (const auto& e : arrive)
            if (e.first.first < hi && lo < e.first.second)
                wait_ext(st, e.second);
    };
    // The rows below the next tile are updated on side lanes, one lane (stream +
    // GEMM workspace) per arrival piece (one piece without host rows): a piece
    // waiting for its rows never holds up the updates of rows already there.
    std::vector<i32> cuts;  // piece q = rows [cuts[q-1], cuts[q]) (cuts[-1] = 0)
    for (const auto& e : arrive)
        if (e.first.first > 0 && (cuts.empty() || e.first.first > cuts.back())) cuts.push_back(e.first.first);
    auto piece_of = [&](i32 row) {
        return (int)(std::upper_bound(cuts.begin(), cuts.end(), row) - cuts.begin());
    };
    const int max_pieces = ntiles + 1;  // a host run cuts at most at every tile
    if ((int)cuts.size() + 1 > max_pieces) throw Error(7 /*RL_EINVAL*/, "too many host pieces");
    if (dry_)
        for (int q = 0; q < max_pieces; ++q) lanes_[kTileLane - q];
    tile_lane_ = &lanes_.at(kTileLane);
    std::vector<std::pair<std::pair<i32, i32>, cudaEvent_t>> side;  // last iteration's pieces
    std::vector<char> used(max_pieces, 0);  // lanes that joined the launch sequence
    auto update_rows = [&](Lane& ln, i32 lo, i32 hi, i32 i0, i32 mm, i32 a) {
        lane_ = &ln;
        swaps_range_on(ln.st, lo, hi - lo, dyn_rp(i0), dyn_rp(a), i0, a);
        trsm_right(lo, hi - lo, i0, mm);
        gemm(lo, hi - lo, i0, a, dyn_rp(a), dyn_c(n_), n_);
        lane_ = nullptr;
    };
    for (i32 i0 = 0; i0 < m_; i0 += g) {
        const i32 mm = std::min(g, m_ - i0), a = i0 + mm;
        node(i0, mm);
        if (!dry_) {
            // rows complete now may go back to the host (see set_host_overlap)
            for (const auto& kv : dones_) {
                const i32 top_end = kv.first.first + kv.first.second / 2;
                if (top_end > i0 && top_end <= a) {
                    flush_swaps();
                    record_ext(kv.second, s_);
                }
            }
            for (const auto& kv : host_out_) {
                if (kv.first.second > i0 && kv.first.second <= a) {
                    flush_swaps();
                    record_ext(kv.second, s_);
                }
            }
        }
        if (a >= m_) break;
        const i32 g2 = std::min(g, m_ - a), b0 = a + g2;
        // the next tile's rows: updated against the tile before by the side lanes
        // (the pieces holding them), possibly still arriving from the host
        for (const auto& sp : side)
            if (!dry_ && sp.first.first < b0 && a < sp.first.second)
                RL_CUDA_CHECK(cudaStreamWaitEvent(s_, sp.second, 0));
        side.clear();
        wait_rows(s_, a, b0);
        swaps_range(a, g2, dyn_rp(i0), dyn_rp(a), i0, a);           // factor.cpp:42
        flush_swaps();
        if (!dry_ && uinv_join_ && !uflags_) {  // the last leaf's U^{-1}
            RL_CUDA_CHECK(cudaStreamWaitEvent(s_, uinv_join_, 0));
            uinv_join_ = nullptr;
        }
        // the next tile: TRSM (factor.cpp:45-46), then the slice its first window
        // reads, the rest of its columns on s2_ (joined before its first tail)
        trsm_end_ = a;
        trsm_right(a, g2, i0, mm);
        gemm(a, g2, i0, a, dyn_rp(a), Dyn{a, PW}, std::min<i64>(PW, n_), s_, n_);
        const cudaEvent_t rest_ev = rest_update(a, g2, i0, a);
        // the rows below the next tile, beside its recursion (each lane FIFO: after
        // the same rows' updates against the earlier tiles); their TRSM may wait
        // for P_j's big inverse (built on inv_lane_) and is one GEMM then
        trsm_end_ = a + 1;
        if (dry_) {
            // size every lane for both layouts: one piece (device input) and one
            // piece per tile (host input)
            events_needed_ += 2 * (max_pieces + 1);
            if (b0 < m_) update_rows(lanes_.at(kTileLane), b0, m_, i0, mm, a);
            for (i32 lo = b0; lo < m_; lo += g)
                update_rows(lanes_.at(kTileLane - std::min(max_pieces - 1, lo / g)), lo, std::min(m_, lo + g), i0,
                            mm, a);
            continue;
        }
        for (i32 lo = b0; lo < m_;) {
            const int q = piece_of(lo);
            const i32 hi = q < (int)cuts.size() ? std::min(m_, cuts[q]) : m_;
            Lane& ln = lanes_.at(kTileLane - q);
            used[q] = 1;
            fork_to(s_, ln.st);
            // ... after the next tile's rest (s2_) has the GPU: the lane's
            // persistent GEMM would otherwise take most SMs first
            if (tile_after_rest_) RL_CUDA_CHECK(cudaStreamWaitEvent(ln.st, rest_ev, 0));
            wait_rows(ln.st, lo, hi);
            update_rows(ln, lo, hi, i0, mm, a);
            cudaEvent_t e = events_.at(next_event_++);
            RL_CUDA_CHECK(cudaEventRecord(e, ln.st));
            side.push_back({{lo, hi}, e});
            lo = hi;
        }
    }
    // The tiles' transpositions onto the U rows of the earlier tiles (the V1
    // swaps of factor.cpp:56 at the tile level), deferred to the end: tile t's U
    // rows are read by nothing after its own iteration, and the transpositions of
    // all later pivots in increasing order are one job per tile (disjoint rows).
    if (dry_) events_needed_ += max_pieces;
    for (int q = 0; q < max_pieces; ++q)
        if (!dry_ && used[q]) fork_to(lanes_.at(kTileLane - q).st, s_);  // their GEMMs read those rows
    for (i32 i0 = 0; i0 + g < m_; i0 += g) {
        const i32 a = i0 + g;
        swaps_gather(dyn_rp(i0), dyn_rp(a), g, dyn_rp(a), dyn_rp(m_), a, m_);
    }
    tiling_ = false;
}

void CupEngine::enqueue(u32* dA, cudaStream_t s) {
    A_ = dA;
    s_ = s;
    stats_ = Stats{};
    swap_jobs_.n = 0;
    ninv_done_.clear();
    next_event_ = 0;
    pending_joins_.clear();
    uinv_join_ = nullptr;
    row_joins_.clear();
    big_ready_.clear();
    lane_ = nullptr;
    early_used_ = false;
    fill_rp0(rp_, s);
    bump_epoch(epoch_, s);  // this run's value of the U^{-1}-ready flags
    if (m_ > 0 && n_ > 0) {
        const bool tl = tiled_on();
        if (tl) tiled(tile_g_);
        else node(0, m_);
        for (cudaEvent_t e : pending_joins_) RL_CUDA_CHECK(cudaStreamWaitEvent(s_, e, 0));
        // (the tile lanes joined s_ at the end of tiled())
        pending_joins_.clear();
        if (m_ > PB && split_max_k_ >= PB) fork_to(s2_, s_);  // s2_ joined the capture at a split
        if (!RL_UINV_IN_TAIL) fork_to(s3_, s_);
        if (!big_ready_.empty()) fork_to(inv_lane_.st, s_);  // the last builds rejoin the capture
        if (early_used_) fork_to(sb_, s_);
        flush_swaps();
        compact_u_rows(A_, lda_, m_, n_, rp_, rrp_, s);
        stats_.launches += 1;
    }
}

void CupEngine::set_host_overlap(const NodeEvents& waits, const NodeEvents& dones) {
    if (waits == waits_ && dones == dones_) return;
    waits_ = waits;
    dones_ = dones;
    if (graph_exec_) {  // the captured sequence no longer matches
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
        graph_A_ = nullptr;
    }
}

void CupEngine::set_host_rows(const RowEvents& in, const RowEvents& out) {
    if (in == host_in_ && out == host_out_) return;
    host_in_ = in;
    host_out_ = out;
    if (graph_exec_) {
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
        graph_A_ = nullptr;
    }
}

void CupEngine::run(u32* dA, cudaStream_t s, bool use_graph) {
    if (!use_graph) {
        enqueue(dA, s);
        RL_CUDA_CHECK(cudaEventRecord(done_, s));
        return;
    }
    if (!graph_exec_ || graph_A_ != dA) {
        if (graph_exec_) {
            cudaGraphExecDestroy(graph_exec_);
            graph_exec_ = nullptr;
        }
        cudaStream_t cs;
        int prio_lo = 0, prio_hi = 0;
        RL_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        RL_CUDA_CHECK(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, prio_hi));
        cudaGraph_t graph;
        RL_CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue(dA, cs);
        } catch (...) {
            cudaStreamEndCapture(cs, &graph);
            cudaStreamDestroy(cs);
            throw;
        }
        RL_CUDA_CHECK(cudaStreamEndCapture(cs, &graph));
        RL_CUDA_CHECK(cudaGraphInstantiate(&graph_exec_, graph, 0));
        RL_CUDA_CHECK(cudaGraphDestroy(graph));
        RL_CUDA_CHECK(cudaStreamDestroy(cs));
        graph_A_ = dA;
    }
    RL_CUDA_CHECK(cudaGraphLaunch(graph_exec_, s));
    RL_CUDA_CHECK(cudaEventRecord(done_, s));
}

void CupEngine::results(i64* rank, u32* rrp_host, u32* ipiv_host, cudaStream_t s) {
    i32 r = 0;
    if (m_ > 0 && n_ > 0) {
        RL_CUDA_CHECK(cudaMemcpyAsync(&r, rp_ + m_, sizeof(i32), cudaMemcpyDeviceToHost, s));
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    *rank = r;
    if (r > 0) {
        if (rrp_host)
            RL_CUDA_CHECK(cudaMemcpyAsync(rrp_host, rrp_, sizeof(i32) * r, cudaMemcpyDeviceToHost, s));
        if (ipiv_host)
            RL_CUDA_CHECK(cudaMemcpyAsync(ipiv_host, ipiv_, sizeof(i32) * r, cudaMemcpyDeviceToHost, s));
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
    }
}

// sigma = identity, then swap(sigma[j], sigma[ipiv[j]]) for j = 0..r-1: the
// composition perm_compose(P2.embed_at(r1,n), P1) of factor.cpp:78-79 unrolled
// over the recursion (perm.cpp:41-79).
void sigma_from_ipiv(i64 n, i64 r, const u32* ipiv, u32* sigma) {
    for (i64 j = 0; j < n; ++j) sigma[j] = (u32)j;
    for (i64 j = 0; j < r; ++j) std::swap(sigma[j], sigma[ipiv[j]]);
}

// Exact OpCounter of the reference cup (field.hpp:16-34) without counting on
// the device: the charges are a pure function of the row-halving skeleton, the
// row profile and the pivot positions.
//   node of R=m-k bottom rows, width w, top rank r1:
//     trsm Right/Upper/Unit: R*r1(r1-1)/2 mul and as many add/sub (kernels.cpp:92-101, 149-154)
//     if r1 < w: Schur mm: R*(w-r1)*r1 mul and as many add/sub (kernels.cpp:54-68)
//     if r1 == w: early return (factor.cpp:47)
//   leaf row (factor.cpp:12-28): pivot j -> (ipiv[j]-j+1) ztest, 1 inv, (w-1) mul;
//     no pivot -> w ztest.
namespace {
struct OpWalk {
    const std::vector<i64>& rpre;  // rank prefix by row
    const u32* ipiv;
    u64 mul = 0, addsub = 0, divinv = 0, ztest = 0;
    void walk(i64 i0, i64 m, i64 w) {
        if (m == 0 || w == 0) return;
        if (m == 1) {
            const i64 j = rpre[i0];
            if (rpre[i0 + 1] > j) {
                ztest += (u64)(ipiv[j] - j + 1);
                divinv += 1;
                mul += (u64)(w - 1);
            } else {
                ztest += (u64)w;
            }
            return;
        }
        const i64 k = m / 2;
        walk(i0, k, w);
        const i64 r1 = rpre[i0 + k] - rpre[i0];
        const i64 R = m - k;
        const u64 t = (u64)R * (u64)r1 * (u64)(r1 > 0 ? r1 - 1 : 0) / 2;
        mul += t;
        addsub += t;
        if (r1 == w) return;
        const u64 s = (u64)R * (u64)(w - r1) * (u64)r1;
        mul += s;
        addsub += s;
        walk(i0 + k, m - k, w - r1);
    }
};
}  // namespace

void cup_opcount(i64 m, i64 n, i64 r, const u32* rrp, const u32* ipiv, u64 ops[4]) {
    std::vector<i64> rpre(m + 1, 0);
    i64 j = 0;
    for (i64 i = 0; i < m; ++i) {
        rpre[i] = j;
        if (j < r && (i64)rrp[j] == i) ++j;
    }
    rpre[m] = j;
    OpWalk w{rpre, ipiv};
    w.walk(0, m, n);
    ops[0] = w.mul;
    ops[1] = w.addsub;
    ops[2] = w.divinv;
    ops[3] = w.ztest;
}

}  // namespace rl
