// cull.cu -- certified tile culling for the global top-K (placeholder: the
// brute-force scan until the certified lists land).
#include "igs_internal.cuh"

int igs_raster_culled(igs_ctx* ctx, int W, int H, int k, int row0, int row1, float* out, uint32_t* topk) {
    return igs_raster_global(ctx, W, H, k, row0, row1, out, topk);
}

int igs_topk_samples_culled(igs_ctx* ctx, const double* uv, uint32_t npts, int k, uint32_t* oi, double* oq) {
    return igs_topk_points(ctx, uv, npts, k, oi, oq);
}

int igs_cull_lists(igs_ctx* ctx, int, int, int, uint32_t*, uint64_t*, uint32_t*, uint32_t*, double*) {
    return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "tile lists not available in this build");
}
