// kernels.cuh -- host launchers of the kernels (each defined and launched in
// its own translation unit; see kernels.cu and cast_curved.cu).
#pragma once
#include "rc_internal.cuh"

namespace rc {

cudaError_t launch_cull(const CamConst& cc, const TreeConst* trees, DevLeafView L, int64_t n, int R, bool affine,
                        int32_t* flag, Rect16* rect, cudaStream_t s);
cudaError_t launch_compact(const int32_t* flag, const Rect16* rect, const int64_t* pos, int64_t n, int32_t* vis,
                           Rect16* vis_rect, cudaStream_t s);
cudaError_t launch_chunk_count(const Rect16* vis_rect, const int64_t* nvis_p, int64_t n, int64_t* cnt,
                               int64_t* counters, cudaStream_t s);
cudaError_t launch_expand(const int64_t* off, const int64_t* nvis_p, int64_t nvis, int32_t* chunk_elem,
                          cudaStream_t s);
cudaError_t launch_cast_affine(const CamConst& cc, const TreeConst* trees, DevLeafView L, int P, const int32_t* vis,
                               const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                               int64_t nchunks, uint32_t key_base, rc_seg* segs, int64_t seg_cap, int32_t* hits_pp,
                               int64_t* counters, int grid, cudaStream_t s, const int64_t* d_nchunks = nullptr);
// surface forests (surface.cu)
cudaError_t launch_cull_surface(const CamConst& cc, const TreeConst* trees, DevLeafView L, int64_t n, int32_t* flag,
                                Rect16* rect, cudaStream_t s);
cudaError_t launch_cast_surface(const CamConst& cc, const TreeConst* trees, DevLeafView L, const int32_t* vis,
                                const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                                int64_t nchunks, uint32_t key_base, rc_seg* segs, int64_t seg_cap, int32_t* hits_pp,
                                int64_t* counters, int grid, cudaStream_t s);
cudaError_t launch_units(const int32_t* vis, const int64_t* nvis_p, int64_t nvis, const int32_t* leaf_node,
                         const int32_t* node_first, const int64_t* chunk_off, int32_t* ucnt, int64_t* uoff,
                         int32_t* uend, int64_t* scan_tmp, uint32_t key_base, Unit* units, bool emit,
                         cudaStream_t s);
cudaError_t launch_cast_curved(const CamConst& cc, const TreeConst* trees, DevLeafView L, int P, const int32_t* vis,
                               const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                               const Unit* units, int64_t nunits, int fold, uint32_t key_base, void* scratch,
                               rc_seg* out, int64_t out_cap, int32_t* hits_pp, int64_t* counters, int grid,
                               const void* gslot, const void* gorg, int64_t v0, int64_t v1, cudaStream_t s);
// element slots of the visible leaves [v0, v1) for the curved segment kernel (slot_record_bytes() each)
cudaError_t launch_prep_slots(const TreeConst* trees, DevLeafView L, int P, const int32_t* vis,
                              const int64_t* nvis_p, int64_t v0, int64_t v1, void* gslot, void* gorg,
                              cudaStream_t s);
size_t slot_record_bytes();
size_t cast_curved_scratch_per_cta();
int cast_curved_ctas_per_sm();
cudaError_t launch_coarsen(const rc_seg* recs, int64_t nrec, int64_t nleaf, const uint32_t* perm, const int64_t* off,
                           int64_t npix,
                           const int32_t* node_first, const int32_t* leaf_node, uint32_t key_base, float tau, rc_seg* out,
                           int64_t out_cap, int32_t* defer, int32_t* mid, int64_t* counters, int max_grid,
                           cudaStream_t s);
cudaError_t launch_pack(const rc_seg* segs, const int64_t* nseg_p, int W, int tw, int th, int tiles_x, int nranks,
                        int64_t* counts, const int64_t* dest_off, int64_t* cursor, rc_seg* out, int grid, bool count,
                        cudaStream_t s);
cudaError_t launch_leaf_weights(const int32_t* flag, const Rect16* rect, int64_t n, int64_t* w, cudaStream_t s);
cudaError_t launch_pack_offsets(const int64_t* counts, int nranks, int64_t* dest_off, cudaStream_t s);
// d_n (optional): the record count read on the device (CUDA-graph frames), n ignored
cudaError_t launch_hist(const rc_seg* segs, int64_t n, int32_t* cnt, int grid, cudaStream_t s,
                        const int64_t* d_n = nullptr);
cudaError_t launch_scatter(const rc_seg* segs, int64_t n, const int64_t* off, int32_t* cursor, uint32_t* out,
                           int grid, cudaStream_t s, const int64_t* d_n = nullptr);
// aggregation: pixel-bucketed permutation (perm, off[npix+1]) by 32-pixel bands; scratch: >= 8 n bytes
cudaError_t launch_band_bucket(const rc_seg* segs, int64_t n, int64_t npix, int32_t* bcnt, int64_t* boff,
                               int64_t* scan_tmp, void* scratch, uint32_t* perm, int64_t* off, int grid,
                               cudaStream_t s);
cudaError_t launch_scatter_rec(const rc_seg* segs, int64_t n, const int64_t* off, int32_t* cursor, rc_seg* out,
                               int grid, cudaStream_t s, const int64_t* d_n = nullptr);
cudaError_t launch_fold(const rc_seg* recs, const uint32_t* perm, const int64_t* off, int W, int H, int tw, int th,
                        const int32_t* my_tiles, int tiles_x, int64_t npix_out, const float bg[3], float tau,
                        float* rgba, int32_t* defer, int64_t* counters, int max_grid, cudaStream_t s);

}  // namespace rc
