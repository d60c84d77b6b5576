// bsp.cu -- BSP partition (placeholder until the shell-binning kernels land).
#include "igs_internal.cuh"

int igs_partition_free(igs_ctx* ctx) { ctx->part = nullptr; return IGS_OK; }

extern "C" {
int igs_partition_build(igs_ctx* ctx, int) { return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "not implemented"); }
int igs_partition_rebuild(igs_ctx* ctx, const double*, uint32_t) { return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "not implemented"); }
int igs_partition_info(igs_ctx* ctx, uint32_t*, uint64_t*) { return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "not implemented"); }
int igs_partition_get(igs_ctx* ctx, double*, double*, uint32_t*, uint32_t*) { return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "not implemented"); }
int igs_locate_blocks(igs_ctx* ctx, const double*, uint32_t, int32_t*) { return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "not implemented"); }
int igs_render_image_blocked(igs_ctx* ctx, int, int, int, float*) { return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "not implemented"); }
int igs_render_points_blocked(igs_ctx* ctx, const double*, uint32_t, int, double*) { return igs_fail(ctx, IGS_E_INVALID_PARAMETER, "not implemented"); }
}
