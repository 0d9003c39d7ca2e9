/*
 * gsparc_b200.h -- C ABI of the B200-native GSpaRC render/train hot path.
 *
 * Plain pointers and sizes only: every pointer argument named *_dev or
 * living inside a frame/cloud struct is DEVICE memory (allocated by the
 * caller, e.g. from PyTorch); `stream` is a cudaStream_t passed as void*.
 * No entry point allocates device memory or synchronises the stream, so the
 * calls can be captured into a CUDA graph.  Every function returns
 * GSPARC_OK (0) or an error code; gsparc_last_error() describes the last
 * failure on the calling thread.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/rfsplat/, see INTEGRATION.md for the bindings):
 *   gsparc_prepare          geometry.cull (geometry.py:198-224) and the
 *                           geometry part of rasterizer._Prepared
 *                           (rasterizer.py:75-102)
 *   gsparc_bin_tiles        np.lexsort depth order (rasterizer.py:82-87) and
 *                           rasterizer._tile_lists (rasterizer.py:115-145)
 *   gsparc_mlp_coef         mlp.direction_angles + mlp.batch_mlp_forward and
 *                           coef = s / d_tx (rasterizer.py:103-111,200;
 *                           mlp.py:40-45,83-89)
 *   gsparc_raster_forward   per-tile compositing do_tile/_tile_alphas
 *                           (rasterizer.py:169-231)
 *   gsparc_render_forward   rasterizer.rasterize_forward
 *                           (rasterizer.py:187-234), batched over TX
 *   gsparc_render_backward  rasterizer.rasterize_backward
 *                           (rasterizer.py:262-378), summed over TX
 *   gsparc_loss_fwd_bwd     image.magnitude/magnitude_backward
 *                           (image.py:46-61) + optimize.combined_loss
 *                           (optimize.py:165-188)
 *   gsparc_adam_step        optimize.adam_step (optimize.py:234-259) with
 *                           optimize.position_lr (optimize.py:205-213)
 *   gsparc_gt_spectrum      rfsim.ground_truth_spectrum (rfsim.py:75-99)
 *                           + free_space_amplitude (rfsim.py:65-71),
 *                           batched over TX
 *   gsparc_rssi_energy      the energy sum of rfsim.rssi_from_spectrum
 *                           (rfsim.py:227-243), batched over images
 */
#ifndef GSPARC_B200_H
#define GSPARC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSPARC_ABI_VERSION 5

enum {
  GSPARC_OK = 0,
  GSPARC_ERR_ARG = 1,         /* invalid argument (shape, null pointer)   */
  GSPARC_ERR_CUDA = 2,        /* CUDA launch / runtime error              */
  GSPARC_ERR_UNSUPPORTED = 3  /* configuration not compiled in            */
};

enum { GSPARC_F32 = 0, GSPARC_F64 = 1 };

/* render flags */
enum {
  GSPARC_LAZY_MLP = 1,    /* evaluate the MLP only for Gaussians with at least
                             one included contribution (exact)            */
  GSPARC_FORCE_FUSED = 2  /* single raster pass even for wide channels     */
};

/* frame counters (int32, at frame + off_counters) */
enum {
  GSPARC_CNT_KEPT = 0,      /* Gaussians kept by the cull                */
  GSPARC_CNT_PAIRS = 1,     /* total (tile, Gaussian) pairs               */
  GSPARC_CNT_OVERFLOW = 2,  /* nonzero: pairs exceeded pair_capacity      */
  GSPARC_CNT_LIVE = 3,      /* Gaussians with >= 1 included contribution  */
  GSPARC_CNT_NONFINITE = 4, /* nonzero: non-finite gradient seen by Adam  */
  GSPARC_CNT_BIGTILE = 5,   /* tiles sorted by the out-of-shared-mem path */
  GSPARC_CNT_SORTED = 6,    /* tiles published to the K3 -> K4a queue     */
  GSPARC_CNT_CLAIMED = 7,   /* queue entries claimed by pass-A CTAs       */
  GSPARC_CNT_PXA_DONE = 8,  /* pass-A CTAs whose live-list entries are written */
  GSPARC_NUM_COUNTERS = 16
};

/* Learnable Gaussian cloud, source order (scene.py:46-103). */
typedef struct gsparc_cloud {
  int64_t n;
  int32_t mlp_in, mlp_hidden, mlp_out; /* (5, 16, 2F) (mlp.py:6-7)        */
  int32_t reserved;
  const double* positions;     /* (n,3) f64                              */
  const double* log_scales;    /* (n,3) f64                              */
  const double* rotations;     /* (n,4) f64, (w,x,y,z), unnormalised      */
  const double* raw_opacities; /* (n)   f64 logits                        */
  const float* mlp_weights;    /* (n,P) f32, W1|b1|W2|b2 rows             */
  const double* mlp_weights64; /* optional (n,P) f64 copy; used by f64
                                  frames (verification path) when non-null */
} gsparc_cloud;

/* Receiver pose + image size (geometry.py:34-47). */
typedef struct gsparc_view {
  double rx[3];
  double rotation[9]; /* row-major W (world -> receiver), orthonormal */
  int32_t width, height;
} gsparc_view;

/* Byte offsets of the per-render device state inside one caller-owned
 * workspace ("frame").  Filled by gsparc_plan_frame. */
typedef struct gsparc_frame_layout {
  int64_t total_bytes;
  int64_t n;              /* Gaussians                                 */
  int64_t pair_capacity;  /* (tile, Gaussian) pair slots               */
  int64_t channels;       /* coef/image channels per pixel, B * C       */
  int32_t width, height, ntx, nty, ntiles, dtype, with_backward, reserved;
  int64_t off_key;        /* u64  [n]   depth key (source order)        */
  int64_t off_rec32;      /* f32  [n,8] raster record                   */
  int64_t off_rec64;      /* f64  [n,8] raster record (dtype f64 only)  */
  int64_t off_rect;       /* i32  [n,4] tile rectangle + pair count     */
  int64_t off_counters;   /* i32  [16]                                  */
  int64_t off_tile_count; /* i32  [ntiles] pairs per tile               */
  int64_t off_tile_cursor;/* i32  [ntiles] K3 -> K4a queue: tile + 1 in sort-completion order (zeroed) */
  int64_t off_tile_start; /* i32  [ntiles+1]                            */
  int64_t off_tile_stop;  /* i32  [ntiles*4] list prefix visited per sub-tile */
  int64_t off_pairs;      /* u64  [pair_capacity] per-tile sorted lists */
  int64_t off_T;          /* dtype[h,w] final transmittance             */
  int64_t off_count;      /* i32  [h,w] contributor count               */
  int64_t off_last;       /* i32  [h,w] end of included list range      */
  int64_t off_live;       /* i32  [n]   Gaussian has >=1 contribution   */
  int64_t off_live_list;  /* i32  [n]   compact live source indices     */
  int64_t off_coef;       /* f32/f64 [n,channels] s/d per Gaussian,TX   */
  int64_t off_gcoef;      /* f32/f64 [n,channels] dL/dcoef (backward)   */
  int64_t off_ggeo;       /* f32/f64 [n,8] dL/d(conic3,mean2d2,sigma)   */
  int64_t off_pair_rec;   /* unused since ABI 2 (0)                       */
  int64_t off_wstop;      /* i32  [ntiles*8] visited list prefix per
                             32-pixel warp (2 rows x 16 px)               */
  int64_t off_rrec;       /* f32  [n,8] f32 raster record {mx,my,qa,qb,
                             qc,opacity,xr,yr} (f32 frames)               */
  int64_t off_ch_idx;     /* u32  [slots,32] per half-tile CTA: source
                             indices of the culled list, 32 per chunk     */
  int64_t off_ch_T;       /* f32  [slots,128] transmittance of the CTA's
                             128 pixels at the start of every chunk       */
  int64_t off_ch_n;       /* i32  [2*ntiles] chunks with a contribution   */
  int64_t off_ch_rec;     /* f32  [slots,32,8] chunk entry records
                             {mx,my,qa,qb,qc,opacity,list pos,index}      */
  int64_t ch_slots;       /* chunk slots (>= 2*(pairs+31*ntiles)/32 + 2) */
  int64_t off_ch_used;    /* u32  [slots] entries of a chunk with at least
                             one included contribution in the CTA        */
  int64_t off_det_gcoef;  /* dtype [pair_capacity,4,channels] per (list
                             entry, sub-tile) dL/dcoef partials
                             (with_backward == 2: deterministic backward) */
  int64_t off_det_ggeo;   /* dtype [pair_capacity,4,max(1,ceil(ch/4)),6]
                             geometric partials (with_backward == 2)      */
  int64_t off_stage;      /* u64  [pair_capacity] unsorted pairs staged
                             by gsparc_prepare, one contiguous segment per
                             (preprocess CTA, tile)                       */
  int64_t off_seg;        /* i32  [ntiles,seg_stride,2] staged segment of
                             preprocess CTA s for tile t: {stage offset,
                             length}, length 0 when the CTA has none      */
  int64_t seg_stride;     /* segment slots per tile (preprocess CTAs)     */
  int64_t off_pxw;        /* f32  [2*ntiles,pxw_chunks,8,128,4] per-pixel
                             blending weights T*alpha (entry quad, pixel,
                             4 entries) of the first pxw_chunks chunks of
                             every half-tile CTA, written by the weights
                             pass (f32 frames)                           */
  int64_t pxw_chunks;     /* chunks per CTA with stored weights          */
  int64_t off_ch_wm;      /* u32  [slots,4] per 32-pixel warp: entries of
                             the chunk with an included contribution     */
  int64_t off_det_inv;    /* i32  [n,320] list position of every (Gaussian,
                             tile of its rectangle) in canonical tile order
                             (with_backward == 2; written by K3)          */
  int64_t off_sort_tmp;   /* u64  [pair_capacity] K3 scratch for tile lists
                             longer than shared memory                    */
  int64_t off_ch_pos;     /* i32  [slots,32] list position (from the tile's
                             start) of every chunk entry, written by the
                             weights pass; the tensor-core raster backward
                             walks only the entries a CTA used (f32
                             frames with a backward; else 0)             */
} gsparc_frame_layout;

int gsparc_abi_version(void);
const char* gsparc_last_error(void);

/* Compute the frame layout for n Gaussians, a width x height image,
 * `channels` = n_tx * mlp_out coef channels and `pair_capacity` pairs. */
int gsparc_plan_frame(int64_t n, int32_t width, int32_t height,
                      int64_t channels, int64_t pair_capacity, int32_t dtype,
                      int32_t with_backward, gsparc_frame_layout* out);

/* K2: cull, radial depth key, equirect projection, pole-clamped Jacobian,
 * 2-D covariance/conic/radii, opacity, tile rectangle (f64 throughout). */
int gsparc_prepare(const gsparc_cloud* cloud, const gsparc_view* view,
                   void* frame, const gsparc_frame_layout* L, void* stream);

/* K3: sort every tile list by (radial depth, source index), bit-exact.
 * gsparc_prepare has already binned the kept Gaussians into 16x16 tiles
 * (incl. the azimuth-seam duplicate) as staged segments; this gathers each
 * tile's segments, sorts them and writes pairs/tile_start. */
int gsparc_bin_tiles(void* frame, const gsparc_frame_layout* L, void* stream);

/* K1: coef[i, b*C + c] = MLP_i(tx_b, theta_i, phi_i)[c] / max(|mu_i-tx_b|, .05)
 * tx_dev: f64 [n_tx,3] device.  live_only: only Gaussians in the live list
 * (requires a preceding weights-only raster pass). */
int gsparc_mlp_coef(const gsparc_cloud* cloud, const double* tx_dev,
                    int32_t n_tx, int32_t live_only, void* frame,
                    const gsparc_frame_layout* L, void* stream);

/* K4: front-to-back compositing.  pass 0 = fused (aux + image),
 * 1 = weights only (aux + live list), 2 = image only (after pass 1).
 * image_out: dtype [n_tx, h, w, C] (ignored for pass 1). */
int gsparc_raster_forward(void* frame, const gsparc_frame_layout* L,
                          int32_t n_tx, int32_t channels_per_tx,
                          double t_eps, int32_t pass, void* image_out,
                          void* stream);

/* K2 + K3 + K1 + K4 in one call (rasterize_forward, batched over TX). */
int gsparc_render_forward(const gsparc_cloud* cloud, const gsparc_view* view,
                          const double* tx_dev, int32_t n_tx, double t_eps,
                          int32_t flags, void* frame,
                          const gsparc_frame_layout* L, void* image_out,
                          void* stream);

/* K5 + K6: gradients of sum_b <dL_b, img_b> w.r.t. every parameter group,
 * written (overwritten) into grad_flat = positions|log_scales|rotations|
 * raw_opacities|mlp_weights, n*(11+P) floats of `grad_dtype`.
 * dL_dev: frame dtype [n_tx, h, w, C].  Requires the matching forward's
 * frame (fused pass, same tx). deterministic: fixed-order reduction (bit-identical reruns); needs a frame
 * planned with with_backward == 2. */
int gsparc_render_backward(const gsparc_cloud* cloud, const gsparc_view* view,
                           const double* tx_dev, int32_t n_tx,
                           const void* dL_dev, int32_t deterministic,
                           void* frame, const gsparc_frame_layout* L,
                           void* grad_flat, int32_t grad_dtype, void* stream);

/* Scratch bytes needed by gsparc_loss_fwd_bwd. */
int64_t gsparc_loss_scratch_bytes(int32_t n_img, int32_t height, int32_t width,
                                  int32_t channels);

/* K7: per image b: pred = |img| (supervision 0, C must be 2) or img
 * (supervision 1); loss = (1-lam) L1 + lam (1 - SSIM) (11x11 Gaussian window,
 * sigma 1.5, reflect padding); dimg = dloss/dimg chained through the
 * magnitude.  img/gt/dimg in `dtype` (GSPARC_F32 / GSPARC_F64); gt has
 * 1 (magnitude) or C channels; arithmetic is f64.
 * stats_out: f64 [n_img, GSPARC_LOSS_STATS] = (loss, l1, ssim, mse,
 * ssim of channel 0, mse of channel 0) per image; the last two are what the
 * reference's train_step logs (optimize.py:281,293). */
#define GSPARC_LOSS_STATS 6
int gsparc_loss_fwd_bwd(const void* img_dev, const void* gt_dev,
                        int32_t dtype, int32_t n_img, int32_t height,
                        int32_t width, int32_t channels, int32_t supervision,
                        double lam, void* dimg_dev, double* stats_out_dev,
                        void* scratch_dev, int64_t scratch_bytes,
                        void* stream);

/* Adam hyper-parameters (optimize.py:27-49). */
typedef struct gsparc_adam_config {
  double position_lr_init, position_lr_final, position_lr_delay_mult;
  double position_lr_max_steps;
  double opacity_lr, scaling_lr, rotation_lr, mlp_lr;
  double beta1, beta2, eps;
} gsparc_adam_config;

/* K8: in-place Adam on the cloud with per-group learning rates and the
 * annealed position schedule; quaternions renormalised afterwards.
 * grad/m/v: f32 flat, layout as grad_flat.  step_dev: int64 device scalar
 * (zero-based iteration, incremented on success).  If any gradient is
 * non-finite nothing is updated and counters_dev[GSPARC_CNT_NONFINITE] is
 * set to 1 + the index of the first bad group (positions = 1 ...). */
int gsparc_adam_step(double* positions, double* log_scales, double* rotations,
                     double* raw_opacities, float* mlp_weights, int64_t n,
                     int32_t mlp_params, const float* grad_flat, float* m_flat,
                     float* v_flat, int64_t* step_dev, int32_t* counters_dev,
                     const gsparc_adam_config* cfg, void* stream);

/* Point emitter of the multipath oracle (rfsim.py:29-38). */
typedef struct gsparc_emitter {
  double position[3];
  double gain_re, gain_im;
  double angular_spread; /* radians, > 0 */
} gsparc_emitter;

/* K9: |field| at every pixel for each TX (rfsim.ground_truth_spectrum),
 * divided by `scale` when scale > 0.  emitters_dev: [n_emitters] device
 * (1..256); rx: host double[3]; tx_dev: f64 [n_tx,3] device;
 * out_dev: out_dtype [n_tx, height, width] device (row 0 = horizon). */
int gsparc_gt_spectrum(const gsparc_emitter* emitters_dev, int32_t n_emitters,
                       const double* rx, double wavelength,
                       const double* tx_dev, int32_t n_tx, int32_t width,
                       int32_t height, double scale, int32_t out_dtype,
                       void* out_dev, void* stream);

/* K10: energy_dev[b] = sum over the selected pixel indices sel_dev[0..n_sel)
 * of re^2 (+ im^2 when channels == 2) of image b, in f64 (the sum of
 * rfsim.rssi_from_spectrum before the 1/fraction and dB steps).
 * img_dev: dtype [n_img, height, width, channels], channels 1 or 2. */
int gsparc_rssi_energy(const void* img_dev, int32_t dtype, int32_t n_img,
                       int32_t height, int32_t width, int32_t channels,
                       const int64_t* sel_dev, int64_t n_sel,
                       double* energy_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GSPARC_B200_H */
