// extern "C" boundary of libgsparc_b200.so (include/gsparc_b200.h).
// Validation + dispatch only; every kernel launch happens on the caller's
// stream, no allocation, no synchronisation (graph-capturable).
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "kernels.cuh"

namespace gs {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return GSPARC_ERR_CUDA;
  }
  return GSPARC_OK;
}

GeoConst make_geo_const(int w, int h) {
  GeoConst g;
  const double pi = 3.141592653589793;  // np.pi
  g.pi = pi;
  g.ca = (double)w / (2.0 * pi);
  g.ce = 2.0 * (double)h / pi;
  g.half_w_over_pi = 0.0;
  g.pole_lim = 89.0 * (pi / 180.0);  // np.deg2rad(89.0)
  g.cos_lim = cos(g.pole_lim);
  g.sin_lim = sin(g.pole_lim);
  g.cos2_lim = g.cos_lim * g.cos_lim;
  g.inv_pi = 1.0 / pi;
  g.w = w;
  g.h = h;
  g.ntx = (w + TILE - 1) / TILE;
  g.nty = (h + TILE - 1) / TILE;
  return g;
}

static int64_t align_up(int64_t v) { return (v + 255) & ~(int64_t)255; }

static int check_cloud(const gsparc_cloud* c) {
  if (!c) {
    set_error("cloud is null");
    return GSPARC_ERR_ARG;
  }
  if (c->n < 0 || (c->n > 0 && (!c->positions || !c->log_scales || !c->rotations ||
                               !c->raw_opacities || !c->mlp_weights))) {
    set_error("cloud: null array pointer");
    return GSPARC_ERR_ARG;
  }
  if (c->mlp_in != 5 || c->mlp_hidden < 1 || c->mlp_hidden > 32 || c->mlp_out < 1) {
    set_error("cloud: unsupported mlp dims (%d,%d,%d)", c->mlp_in, c->mlp_hidden, c->mlp_out);
    return GSPARC_ERR_UNSUPPORTED;
  }
  if (c->n > 0x7fffffffLL) {
    set_error("cloud: n exceeds 2^31-1");
    return GSPARC_ERR_ARG;
  }
  return GSPARC_OK;
}

static int check_frame(const void* frame, const gsparc_frame_layout* L) {
  if (!frame || !L) {
    set_error("frame or layout is null");
    return GSPARC_ERR_ARG;
  }
  return GSPARC_OK;
}

}  // namespace gs

namespace gs {
extern long long* gsparc_dbg_ptr;
}

using namespace gs;

extern "C" {

int gsparc_abi_version(void) { return GSPARC_ABI_VERSION; }

// experiments only (not in the public header): device pointer of the last
// pass-B timing buffer when GSPARC_PXB_DBG is set
void* gsparc_debug_timing(void) { return (void*)gs::gsparc_dbg_ptr; }
int gsparc_debug_copy(long long* host, int64_t count) {
  if (!gs::gsparc_dbg_ptr) return GSPARC_ERR_ARG;
  return cudaMemcpy(host, gs::gsparc_dbg_ptr, sizeof(long long) * count, cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? GSPARC_OK
             : GSPARC_ERR_CUDA;
}

const char* gsparc_last_error(void) { return g_err; }

int gsparc_plan_frame(int64_t n, int32_t width, int32_t height, int64_t channels,
                        int64_t pair_capacity, int32_t dtype, int32_t with_backward,
                        gsparc_frame_layout* out) {
  if (!out || n < 0 || width < 1 || height < 1 || channels < 1 || pair_capacity < 1 ||
      (dtype != GSPARC_F32 && dtype != GSPARC_F64)) {
    set_error("plan_frame: invalid arguments");
    return GSPARC_ERR_ARG;
  }
  if (pair_capacity > 0x7fffffffLL) {
    set_error("plan_frame: pair_capacity exceeds 2^31-1");
    return GSPARC_ERR_ARG;
  }
  gsparc_frame_layout L;
  memset(&L, 0, sizeof(L));
  L.n = n;
  L.pair_capacity = pair_capacity;
  L.channels = channels;
  L.width = width;
  L.height = height;
  L.ntx = (width + TILE - 1) / TILE;
  L.nty = (height + TILE - 1) / TILE;
  L.ntiles = L.ntx * L.nty;
  L.dtype = dtype;
  L.with_backward = with_backward;
  const int64_t esz = dtype == GSPARC_F64 ? 8 : 4;
  const int64_t nn = n > 0 ? n : 1;
  const int64_t px = (int64_t)width * height;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    int64_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  // counters, tile_count and tile_cursor are contiguous: gsparc_prepare
  // zeroes them with one memset
  L.off_counters = take(sizeof(int) * GSPARC_NUM_COUNTERS);
  L.off_tile_count = take(sizeof(int) * L.ntiles);
  L.off_tile_cursor = take(sizeof(int) * L.ntiles);
  L.off_key = take(8 * nn);
  L.off_rec32 = take(32 * nn);
  L.off_rec64 = take(dtype == GSPARC_F64 ? 64 * nn : 0);
  L.off_rect = take(16 * nn);
  L.off_tile_start = take(sizeof(int) * (L.ntiles + 1));
  L.off_tile_stop = take(sizeof(int) * L.ntiles * 4);  // per sub-tile
  L.off_pairs = take(8 * pair_capacity);
  L.off_T = take(esz * px);
  L.off_count = take(sizeof(int) * px);
  L.off_last = take(sizeof(int) * px);
  L.off_live = take(sizeof(int) * nn);
  L.off_live_list = take(sizeof(int) * nn);
  L.off_coef = take(esz * nn * channels);
  L.off_gcoef = with_backward ? take(esz * nn * channels) : 0;
  L.off_ggeo = with_backward ? take(esz * nn * 8) : 0;
  L.off_pair_rec = 0;
  L.off_wstop = take(sizeof(int) * L.ntiles * 8);
  // f32 raster (raster_px.cu): records + per half-tile chunk lists and
  // transmittance checkpoints.  A CTA's chunks never exceed ceil(len/32),
  // so 2 * floor((tile_start + 31 t) / 32) is a valid per-tile slot base.
  L.ch_slots = 2 * ((pair_capacity + 31 * (int64_t)L.ntiles) / 32) + 2 * L.ntiles + 2;
  L.off_rrec = take(dtype == GSPARC_F32 ? 32 * nn : 0);
  L.off_ch_idx = take(dtype == GSPARC_F32 ? 4 * 32 * L.ch_slots : 0);
  L.off_ch_T = take(dtype == GSPARC_F32 ? 4 * 128 * L.ch_slots : 0);
  L.off_ch_n = take(sizeof(int) * 2 * L.ntiles);
  L.off_ch_rec = take(dtype == GSPARC_F32 ? 32 * 32 * L.ch_slots : 0);
  L.off_ch_used = take(dtype == GSPARC_F32 ? 4 * L.ch_slots : 0);
  const bool det = with_backward == 2;
  const int64_t det_chunks = channels >= 4 ? (channels + 3) / 4 : 1;
  L.off_det_gcoef = det ? take(esz * pair_capacity * 4 * channels) : 0;
  L.off_det_ggeo = det ? take(esz * pair_capacity * 4 * det_chunks * 6) : 0;
  L.seg_stride = (nn + PREP_G - 1) / PREP_G;
  L.off_stage = take(8 * pair_capacity);
  L.off_seg = take(8 * (int64_t)L.ntiles * L.seg_stride);
  L.pxw_chunks = dtype == GSPARC_F32 ? PXW_CHUNKS : 0;
  if (const char* e = getenv("GSPARC_PXW_CHUNKS")) {  // tests: force the recompute path
    const int v = atoi(e);
    if (v >= 0 && v < L.pxw_chunks) L.pxw_chunks = v;
  }
  L.off_pxw = take(4 * 2 * (int64_t)L.ntiles * L.pxw_chunks * 128 * 32);
  L.off_ch_wm = take(dtype == GSPARC_F32 ? 4 * 4 * L.ch_slots : 0);
  // a Gaussian's rectangle covers at most nty rows x ntx columns (the wrap
  // segment never adds columns beyond ntx), so ntiles slots always suffice
  L.off_det_inv = det ? take(sizeof(int) * nn * (int64_t)L.ntiles) : 0;
  L.off_sort_tmp = take(8 * pair_capacity);
  L.off_ch_pos = dtype == GSPARC_F32 && with_backward ? take(4 * 32 * L.ch_slots) : 0;
  L.total_bytes = o;
  *out = L;
  return GSPARC_OK;
}

int gsparc_prepare(const gsparc_cloud* cloud, const gsparc_view* view, void* frame,
                   const gsparc_frame_layout* L, void* stream) {
  GS_TRY(check_cloud(cloud));
  GS_TRY(check_frame(frame, L));
  if (!view || view->width != L->width || view->height != L->height || cloud->n != L->n) {
    set_error("prepare: view/cloud do not match the frame layout");
    return GSPARC_ERR_ARG;
  }
  return launch_preprocess(*cloud, *view, *L, (char*)frame, (cudaStream_t)stream);
}

int gsparc_bin_tiles(void* frame, const gsparc_frame_layout* L, void* stream) {
  GS_TRY(check_frame(frame, L));
  return launch_bin_tiles(*L, (char*)frame, (cudaStream_t)stream);
}

int gsparc_mlp_coef(const gsparc_cloud* cloud, const double* tx_dev, int32_t n_tx,
                    int32_t live_only, void* frame, const gsparc_frame_layout* L, void* stream) {
  GS_TRY(check_cloud(cloud));
  GS_TRY(check_frame(frame, L));
  if (!tx_dev || n_tx < 1) {
    set_error("mlp_coef: need at least one transmitter");
    return GSPARC_ERR_ARG;
  }
  return launch_mlp(*cloud, tx_dev, n_tx, live_only != 0, *L, (char*)frame,
                    (cudaStream_t)stream);
}

int gsparc_raster_forward(void* frame, const gsparc_frame_layout* L, int32_t n_tx,
                          int32_t channels_per_tx, double t_eps, int32_t pass, void* image_out,
                          void* stream) {
  GS_TRY(check_frame(frame, L));
  if (pass < 0 || pass > 2 || n_tx < 1 || channels_per_tx < 1 ||
      (pass != 1 && !image_out)) {
    set_error("raster_forward: invalid arguments");
    return GSPARC_ERR_ARG;
  }
  return launch_raster_forward(*L, (char*)frame, n_tx, channels_per_tx, t_eps, pass, image_out,
                               (cudaStream_t)stream);
}

int gsparc_render_forward(const gsparc_cloud* cloud, const gsparc_view* view,
                          const double* tx_dev, int32_t n_tx, double t_eps, int32_t flags,
                          void* frame, const gsparc_frame_layout* L, void* image_out,
                          void* stream) {
  GS_TRY(check_cloud(cloud));
  GS_TRY(check_frame(frame, L));
  if (!image_out || !tx_dev || n_tx < 1) {
    set_error("render_forward: invalid arguments");
    return GSPARC_ERR_ARG;
  }
  if ((int64_t)n_tx * cloud->mlp_out > L->channels) {
    set_error("render_forward: n_tx*mlp_out exceeds the frame's channels");
    return GSPARC_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* f = (char*)frame;
  GS_TRY(gsparc_prepare(cloud, view, frame, L, stream));
  const bool lazy = (flags & GSPARC_LAZY_MLP) && !(flags & GSPARC_FORCE_FUSED);
  GS_TRY(launch_bin_tiles(*L, f, st, lazy));
  if (lazy) {
    GS_TRY(launch_raster_forward(*L, f, n_tx, cloud->mlp_out, t_eps, 1, image_out, st));
    // f32 frames: the MLP streams the live list while pass A finishes
    const int stream_ctas = L->dtype == GSPARC_F32 ? 2 * (int)L->ntiles : 0;
    GS_TRY(launch_mlp(*cloud, tx_dev, n_tx, true, *L, f, st, stream_ctas));
    return launch_raster_forward(*L, f, n_tx, cloud->mlp_out, t_eps, 2, image_out, st);
  }
  GS_TRY(launch_mlp(*cloud, tx_dev, n_tx, false, *L, f, st));
  return launch_raster_forward(*L, f, n_tx, cloud->mlp_out, t_eps, 0, image_out, st);
}

int gsparc_render_backward(const gsparc_cloud* cloud, const gsparc_view* view,
                           const double* tx_dev, int32_t n_tx, const void* dL_dev,
                           int32_t deterministic, void* frame, const gsparc_frame_layout* L,
                           void* grad_flat, int32_t grad_dtype, void* stream) {
  GS_TRY(check_cloud(cloud));
  GS_TRY(check_frame(frame, L));
  if (!L->with_backward || !dL_dev || !grad_flat || !tx_dev || n_tx < 1) {
    set_error("render_backward: invalid arguments (frame needs with_backward)");
    return GSPARC_ERR_ARG;
  }
  if (deterministic && L->with_backward != 2) {
    set_error("render_backward: deterministic mode needs a frame planned with with_backward=2");
    return GSPARC_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* f = (char*)frame;
  GS_TRY(launch_raster_backward(*L, f, n_tx, cloud->mlp_out, dL_dev, deterministic != 0, st));
  return launch_gauss_backward(*cloud, *view, tx_dev, n_tx, *L, f, grad_flat, grad_dtype, st);
}

int64_t gsparc_loss_scratch_bytes(int32_t n_img, int32_t height, int32_t width,
                                  int32_t channels) {
  return loss_scratch_bytes(n_img, height, width, channels);
}

int gsparc_loss_fwd_bwd(const void* img_dev, const void* gt_dev, int32_t dtype, int32_t n_img,
                        int32_t height, int32_t width, int32_t channels, int32_t supervision,
                        double lam, void* dimg_dev, double* stats_out_dev, void* scratch_dev,
                        int64_t scratch_bytes, void* stream) {
  if (!img_dev || !gt_dev || !dimg_dev || !stats_out_dev || !scratch_dev || n_img < 1 ||
      channels < 1 || (supervision != 0 && supervision != 1) ||
      (dtype != GSPARC_F32 && dtype != GSPARC_F64)) {
    set_error("loss_fwd_bwd: invalid arguments");
    return GSPARC_ERR_ARG;
  }
  return launch_loss(img_dev, gt_dev, dtype, n_img, height, width, channels, supervision, lam,
                     dimg_dev, stats_out_dev, scratch_dev, scratch_bytes, (cudaStream_t)stream);
}

int gsparc_adam_step(double* positions, double* log_scales, double* rotations,
                     double* raw_opacities, float* mlp_weights, int64_t n, int32_t mlp_params,
                     const float* grad_flat, float* m_flat, float* v_flat, int64_t* step_dev,
                     int32_t* counters_dev, const gsparc_adam_config* cfg, void* stream) {
  if (!positions || !log_scales || !rotations || !raw_opacities || !mlp_weights || !grad_flat ||
      !m_flat || !v_flat || !step_dev || !counters_dev || !cfg || n < 0 || mlp_params < 1) {
    set_error("adam_step: invalid arguments");
    return GSPARC_ERR_ARG;
  }
  return launch_adam(positions, log_scales, rotations, raw_opacities, mlp_weights, n, mlp_params,
                     grad_flat, m_flat, v_flat, step_dev, counters_dev, *cfg,
                     (cudaStream_t)stream);
}

int gsparc_gt_spectrum(const gsparc_emitter* emitters_dev, int32_t n_emitters, const double* rx,
                       double wavelength, const double* tx_dev, int32_t n_tx, int32_t width,
                       int32_t height, double scale, int32_t out_dtype, void* out_dev,
                       void* stream) {
  return launch_gt_spectrum(emitters_dev, n_emitters, rx, wavelength, tx_dev, n_tx, width, height,
                            scale, out_dtype, out_dev, (cudaStream_t)stream);
}

int gsparc_rssi_energy(const void* img_dev, int32_t dtype, int32_t n_img, int32_t height,
                       int32_t width, int32_t channels, const int64_t* sel_dev, int64_t n_sel,
                       double* energy_dev, void* stream) {
  return launch_rssi_energy(img_dev, dtype, n_img, height, width, channels, sel_dev, n_sel,
                            energy_dev, (cudaStream_t)stream);
}

}  // extern "C"
