// cup.h -- the device-resident CUP engine (host side).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <set>
#include <unordered_map>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace rl {

struct PanelScratch;

class CupEngine {
public:
    struct Stats {
        long gemms = 0, tc_gemms = 0, panels = 0, trsm_leaves = 0, launches = 0;
    };

    CupEngine(i32 m, i32 n, i64 lda, u32 p);
    ~CupEngine();
    CupEngine(const CupEngine&) = delete;
    CupEngine& operator=(const CupEngine&) = delete;

    // Enqueue the full factorization of the device matrix dA (m x n, lda) on s.
    // With use_graph the launch sequence is captured once per dA and replayed.
    void run(u32* dA, cudaStream_t s, bool use_graph);
    // rank (sync), then row profile / pivot positions (int32 on device) to host.
    void results(i64* rank, u32* rrp_host, u32* ipiv_host, cudaStream_t s);

    const Stats& stats() const { return stats_; }
    i32 m() const { return m_; }
    i32 n() const { return n_; }
    i64 lda() const { return lda_; }
    u32 p() const { return p_; }
    int limbs() const { return L_; }
    size_t workspace_bytes() const { return a2_cap_ + b2_cap_; }
    void set_use_tc(bool v) { use_tc_ = v; }
    // Host-buffer path (PCIe overlapped with the factorization).  waits: node
    // (i0, mm) -> event the launch sequence waits on right after that node's top
    // half, before it first touches the node's bottom rows (they may still be
    // arriving from the host).  dones: node -> event recorded once the node's
    // top half is factored (its rows may go back to the host while the rest
    // runs; valid when no later transposition or U-row move reaches them --
    // sigma and the row profile are the identity -- which the caller checks).
    // Captured as external event nodes: the events must outlive the graph.
    using NodeEvents = std::map<std::pair<i32, i32>, cudaEvent_t>;
    void set_host_overlap(const NodeEvents& waits, const NodeEvents& dones);
    // The same at tile granularity (tiled engines, tile_rows() > 0): in = rows
    // [lo, hi) -> event recorded once they are in device memory (rows below the
    // first lo are resident at launch); out = rows [lo, hi) -> event the launch
    // sequence records once they are factored (same validity rule as dones).
    using RowEvents = std::vector<std::pair<std::pair<i32, i32>, cudaEvent_t>>;
    void set_host_rows(const RowEvents& in, const RowEvents& out);
    i32 tile_rows() const { return tiled_on() ? tile_g_ : 0; }

private:
    void enqueue(u32* dA, cudaStream_t s);
    void node(i32 i0, i32 m);
    // Tiled top level (right-looking over row tiles of tile_g_ rows, each tile
    // factored by node()): see cup.cu
    void tiled(i32 g);
    void panel(i32 i0, i32 b);
    void trsm_right(i32 r0, i32 M, i32 x0, i32 mx);
    void gemm_ninv(i32 r0, i32 M, i32 x0, i32 mx, const u32* ninv, i32 ldn = NINV_LD);
    // big node inverses (nodes of (8, 16] leaves): built on a side lane right
    // after the node is factored, used by the tall TRSMs of the levels above
    void build_big_inverse(i32 x0, i32 mm);
    void combine_inverse(const u32* Xa, i32 la, i32 xa, i32 ma, const u32* Xb, i32 lb, i32 xb, i32 mb, u32* X,
                         i32 ldx, cudaStream_t st);
    void gemm_dense(const u32* A, i64 lda, bool a_dense, const u32* B, i64 ldb, bool b_dense, const i32* gather,
                    u32* C, i64 ldc, i32 M, Dyn k_lo, Dyn k_hi, Dyn n_lo, Dyn n_hi, i64 Kmax, i64 Nmax, u32 alpha,
                    cudaStream_t st);
    // a B operand packed ahead of its GEMM (early_pack_b) and its ready event
    struct EarlyPack {
        uint8_t* buf = nullptr;
        cudaEvent_t ev = nullptr;
    };
    void gemm(i32 row0, i32 M, i32 x0, i32 x1, Dyn n_lo, Dyn n_hi, i64 Nmax, cudaStream_t st = nullptr,
              i32 n_cap = 0, const EarlyPack* ep = nullptr);
    EarlyPack early_pack_b(i32 i0, i32 k, i32 mm);
    cudaEvent_t fork_to(cudaStream_t from, cudaStream_t to);  // `to` waits for `from`'s work so far
    void record_ext(cudaEvent_t e, cudaStream_t st);
    void wait_ext(cudaStream_t st, cudaEvent_t e);
    // the transpositions are the pivots of rows [piv_lo, piv_hi) (whole leaves)
    void swaps_range(i32 row0, i32 M, Dyn j_lo, Dyn j_hi, i32 piv_lo, i32 piv_hi);
    void swaps_range_on(cudaStream_t st, i32 row0, i32 M, Dyn j_lo, Dyn j_hi, i32 piv_lo, i32 piv_hi);
    void swaps_gather(Dyn g_lo, Dyn g_hi, i32 Mmax, Dyn j_lo, Dyn j_hi, i32 piv_lo, i32 piv_hi);
    void leaf_range(i32 piv_lo, i32 piv_hi, SwapArgs& a) const;
    void queue_swaps(const SwapArgs& a);
    void flush_swaps();

    i32 m_, n_;
    i64 lda_;
    u32 p_;
    Fp f_;
    int L_;
    bool dry_ = false;
    bool use_tc_ = true;
    bool fused_trsm_ = true;
    u32* A_ = nullptr;
    cudaStream_t s_ = nullptr;
    // side streams of the captured DAG: s2_ runs the wide part of each Schur
    // update while the next leaf's window kernel runs on s_; s3_ runs each
    // leaf's U^{-1} beside its tail
    cudaStream_t s2_ = nullptr, s3_ = nullptr;
    std::vector<cudaEvent_t> events_;
    size_t next_event_ = 0, events_needed_ = 0;
    std::vector<cudaEvent_t> pending_joins_;   // joined before the next tail
    cudaEvent_t uinv_join_ = nullptr;          // last leaf's U^{-1}, joined before the next TRSM
    SwapJobs swap_jobs_{};                     // queued, launched by flush_swaps()
    // Schur updates with K <= this are split (window slice first, rest on s2_);
    // above it the extra narrow GEMM costs more than the overlap wins
#ifndef RL_SPLIT_MAX_K
#define RL_SPLIT_MAX_K 1024
#endif
    i32 split_max_k_ = RL_SPLIT_MAX_K;
    NodeEvents waits_, dones_;
    RowEvents host_in_, host_out_;
    void* meta_ = nullptr;                     // one allocation for everything below
    i32* rp_ = nullptr;
    i32* rrp_ = nullptr;
    i32* ipiv_ = nullptr;
    PanelScratch* ps_ = nullptr;
    u32* uinv_ = nullptr;                      // one PB x PB block per leaf
    uint16_t* inv_table_ = nullptr;            // p < 2^16: x -> x^{-1} mod p
    std::unordered_map<i32, i32> leaf_of_;     // leaf start row -> leaf index
    std::vector<i32> leaf_starts_;             // leaf start rows, increasing (index order)
    i32* swapflags_ = nullptr;                 // per leaf: made a transposition
    // per leaf: U^{-1} written (== *epoch_, bumped at the start of every run);
    // with uflags_ the bridge and the node TRSM wait on these on the device
    // instead of the critical stream waiting for the U^{-1} kernel's event
#ifndef RL_UREADY
#define RL_UREADY 1
#endif
    i32* uready_ = nullptr;
    i32* epoch_ = nullptr;
    bool uflags_ = false;
    // node inverses U_X^{-1} of <= 4-leaf skeleton nodes X = (x0, mx): computed by
    // the first TRSM against X (as a by-product of its sweep), then reused by the
    // taller TRSMs above as one tensor-core GEMM each
    std::map<std::pair<i32, i32>, i32> ninv_slot_;
    std::set<std::pair<i32, i32>> ninv_done_;  // during one enqueue
    u32* ninv_ = nullptr;
#ifndef RL_NINV_GEMM_MIN_ROWS
#define RL_NINV_GEMM_MIN_ROWS 512
#endif
    static constexpr i32 kNinvGemmMinRows = RL_NINV_GEMM_MIN_ROWS;  // taller G: tensor-core GEMM
    uint8_t* a2_ = nullptr;
    uint8_t* b2_ = nullptr;
    size_t a2_cap_ = 0, b2_cap_ = 0;
    // Row-split of the wide nodes (k > split_max_k_): the TRSM + Schur update of
    // the bottom half's LOWER rows [b0 + bm/2, b0 + bm) is first read after the
    // bottom half's own top half is factored, so it runs on a low-priority side
    // lane (one stream + GEMM workspace per node height) beside that recursion
    // and is joined right before the child node first touches those rows.
#ifndef RL_ROW_SPLIT_MIN_ROWS
#define RL_ROW_SPLIT_MIN_ROWS 4096
#endif
    i32 row_split_min_ = RL_ROW_SPLIT_MIN_ROWS;  // 0: off
    // geometric row split (node()): every bottom half is updated piece by piece
    // in the order the recursion below first touches its rows
#ifndef RL_GEO_SPLIT
#define RL_GEO_SPLIT 0
#endif
    bool geo_split_ = RL_GEO_SPLIT != 0;
#ifndef RL_GEO_MAX_K
#define RL_GEO_MAX_K 512
#endif
    i32 geo_max_k_ = RL_GEO_MAX_K;  // only nodes whose top half has at most this many rows
#ifndef RL_BRIDGE
#define RL_BRIDGE 1
#endif
    bool bridge_on_ = RL_BRIDGE != 0;  // leaf pairs: swaps + TRSM + slice update fused (bridge.cu)
#ifndef RL_LANE_PRIO
#define RL_LANE_PRIO 1
#endif
    bool lane_prio_ = RL_LANE_PRIO != 0;  // lane stream priority by height (else all lowest)
#ifndef RL_LANE_CTAS
#define RL_LANE_CTAS 110
#endif
    i32 lane_ctas_ = RL_LANE_CTAS;               // persistent GEMM CTAs on a lane (0: all but one SM);
                                                 // the rest stay free for the recursion beside it
    struct Lane {
        cudaStream_t st = nullptr;
        uint8_t* a2 = nullptr;
        uint8_t* b2 = nullptr;
        size_t a2_cap = 0, b2_cap = 0;
    };
    std::map<i32, Lane> lanes_;                  // node height bm -> lane
    Lane* lane_ = nullptr;                       // non-null while enqueueing side work
    std::map<std::pair<i32, i32>, cudaEvent_t> row_joins_;  // child node -> side work done
    cudaStream_t work_stream() const { return lane_ ? lane_->st : s_; }
#ifndef RL_BIG_INV
#define RL_BIG_INV 1
#endif
    static constexpr i32 BIG_LD = 16 * PB;         // 1024: pitch of a big node inverse
    static constexpr i32 CH_LD = 8 * PB;           // 512: a child's inverse / the T blocks
#ifndef RL_BIG_MIN_ROWS
#define RL_BIG_MIN_ROWS 2048
#endif
    static constexpr i32 kBigMinRows = RL_BIG_MIN_ROWS;  // TRSMs at least this tall use them
    bool big_on_ = RL_BIG_INV != 0;
    i32 trsm_end_ = 0;  // end row of the triangle the current node's TRSMs solve against
    std::map<std::pair<i32, i32>, i32> big_slot_;          // node -> slot (dry run)
    std::map<std::pair<i32, i32>, cudaEvent_t> big_ready_; // node -> built (one enqueue)
    u32* big_ = nullptr;                                   // BIG_LD x BIG_LD per slot
    u32* big_tmp_ = nullptr;                               // 4 x 256^2 + 4 x 512^2 scratch
    Lane inv_lane_;                                        // stream + GEMM workspace of the builds
    // Early B packs.  The Schur update of a node whose top half has more than
    // split_max_k_ rows reads the top half's U rows as B; they are final once
    // the top half is factored, so their limb image is packed on a side stream
    // right then, beside the TRSM, instead of on the critical path after it
    // (and once for the critical and the row-split lane GEMM together).  One
    // workspace per node height: all GEMMs of a node finish inside the node.
#ifndef RL_EARLY_B
#define RL_EARLY_B 1
#endif
    bool early_b_on_ = RL_EARLY_B != 0;
    struct EarlyBuf {
        uint8_t* buf = nullptr;
        size_t cap = 0;
    };
    std::map<i32, EarlyBuf> early_;              // node height -> B image workspace
    cudaStream_t sb_ = nullptr;                  // the B-pack stream
    bool early_used_ = false;                    // during one enqueue
    // Tiled top level: matrices with tile_min_m_ <= m <= tile_max_m_ rows are
    // factored tile by tile (tiles of tile_g_ rows); 0 disables.
#ifndef RL_TILE_G
#define RL_TILE_G 1024
#endif
#ifndef RL_TILE_MIN_M
#define RL_TILE_MIN_M 4096
#endif
#ifndef RL_TILE_MAX_M
#define RL_TILE_MAX_M 16384
#endif
    i32 tile_g_ = RL_TILE_G, tile_min_m_ = RL_TILE_MIN_M, tile_max_m_ = RL_TILE_MAX_M;
    bool tiled_on() const { return tile_g_ > 0 && m_ >= tile_min_m_ && m_ <= tile_max_m_ && m_ > tile_g_; }
    static constexpr i32 kTileLane = -1;         // lanes_ key of the tiles' side lane
    bool tiling_ = false;                        // inside tiled()
#ifndef RL_TILE_CTAS
#define RL_TILE_CTAS 100
#endif
    i32 tile_ctas_ = RL_TILE_CTAS;               // persistent GEMM CTAs of the tiles' side lane
    Lane* tile_lane_ = nullptr;
    // tile lanes: lanes_ keys kTileLane, kTileLane - 1, ... (one per host-arrival piece)
    bool is_tile_lane(const Lane* l) const {
        if (!l) return false;
        for (const auto& kv : lanes_)
            if (kv.first <= kTileLane && &kv.second == l) return true;
        return false;
    }
    bool tile_after_rest_ = true;                // the lane starts after the next tile's rest GEMM
#ifndef RL_REST_PIECES
#define RL_REST_PIECES 0
#endif
    // (measured slower: C3 24.2 vs 21.6 ms -- the bridge then waits for its piece)
    bool rest_pieces_ = RL_REST_PIECES != 0;     // rest_update() in left-spine pieces
#ifndef RL_REST_SPLIT
#define RL_REST_SPLIT 0
#endif
    // (measured, bit-exact: C3 20.30 ms (1: both GEMMs on s2_) / 20.52 ms (2: the second on a lane) vs 20.13 ms)
    int rest_split_ = RL_REST_SPLIT;             // rest_update(): the first leaf pair's rows first, B packed once
    cudaEvent_t rest_update(i32 b0, i32 bm, i32 x0, i32 x1);
#ifndef RL_S2_PRIO
#define RL_S2_PRIO 0
#endif
    bool s2_prio_ = RL_S2_PRIO != 0;             // s2_ above the lanes at the CTA scheduler
    BridgeArgs leaf_bridge(i32 leaf, i32 leaf_end, i32 row0, i32 M, Dyn n_lo) const;
    cudaGraphExec_t graph_exec_ = nullptr;
    u32* graph_A_ = nullptr;
    cudaEvent_t done_ = nullptr;  // end of the last run: the destructor waits for it
    Stats stats_;
};

void sigma_from_ipiv(i64 n, i64 r, const u32* ipiv, u32* sigma);
void cup_opcount(i64 m, i64 n, i64 r, const u32* rrp, const u32* ipiv, u64 ops[4]);

}  // namespace rl
