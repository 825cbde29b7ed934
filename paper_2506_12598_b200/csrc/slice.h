// slice.h — the SLICE engine (DESIGN.md §4 K3/K4).
//
// For linear slowdown modes every overlap O_w depends on the tuple only through
// (T' = sum_w S'_w, S'_w), so the candidates split into T'-slices and, inside a slice,
// the objective is a (min,+) (SUM) or (min,max) (MAX, ENERGY) knapsack over workers.
//   pass 1  (K3) FP32 suffix DP per slice -> J32(T') (a filter: <= delta from exact)
//   pass 2a exact integer DP on the slices with J32 <= band bound -> exact J(T'), H*
//   pass 2b exact DP + lexicographic walk (K4) on the slices with J within tolerance;
//           each slice's lexicographically smallest qualifying tuple -> global min index.
#pragma once
#include <vector>

#include "engine.h"

namespace eclip {

struct SliceDev {
    int32_t W, Lmax, mode, obj;
    int64_t gS;                 // gcd of every S' (slice step)
    int64_t Tlo, Thi;           // slice range in gS units
    int64_t n_slices;
    int32_t smin[MAXW], smax[MAXW];    // per worker, gS units
    int64_t plo[MAXW + 1], phi[MAXW + 1];  // prefix sums of smin / smax over workers 0..w-1
    int64_t slo[MAXW + 1], shi[MAXW + 1];  // suffix sums over workers w..W-1
    int32_t doff[MAXW];         // offset of worker w's dense map
    int32_t maxrange;           // max D range length
    int32_t pad;                // +inf padding of the FP32 D buffers (max level span + RB)
    int32_t gtot;               // total dense entries
    int32_t shard, n_shards;
    uint64_t tol_num, tol_den;
    double delta;
};

struct SliceState {
    SliceDev h{};
    int16_t* dense = nullptr;       // [gtot] level index per S' offset, -1 if none
    float* J32 = nullptr;           // [n_slices]
    U256* Jex = nullptr;            // [n_slices]
    int32_t* band = nullptr;        // [n_slices] compacted slice list
    int32_t* nband = nullptr;       // [1]
    U256* wtup = nullptr;           // [n_slices] per band slice: its lexmin qualifying tuple (packed)
    uint64_t* scratch = nullptr;    // exact DP tables, per CTA slot
    int32_t slots = 0;
    unsigned long long* d_units = nullptr;  // lattice points of pass 1 (this shard)
    std::vector<void*> allocs;
    cudaStream_t st = nullptr;
    void release();
    ~SliceState();
};

cudaError_t slice_setup(SliceState& s, const Setup& su, const Tables& tb, Work& wk, const int32_t* tabL,
                        const int32_t* table_of, cudaStream_t st);
cudaError_t slice_pass1(SliceState& s, const Setup& su, const Tables& tb, Work& wk, cudaStream_t st);
cudaError_t slice_pass2_min(SliceState& s, const Setup& su, const Tables& tb, Work& wk, cudaStream_t st);
cudaError_t slice_pass2_first(SliceState& s, const Setup& su, const Tables& tb, Work& wk, cudaStream_t st);
cudaError_t slice_decode_winner(SliceState& s, const Setup& su, Work& wk, cudaStream_t st);
uint64_t slice_units(const SliceState& s);

}  // namespace eclip
