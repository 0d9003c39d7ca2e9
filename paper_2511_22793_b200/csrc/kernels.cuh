// Host-side launchers for the K1..K8 kernels (defined in the .cu files).
#pragma once
#include "common.cuh"

namespace gs {

GeoConst make_geo_const(int w, int h);
int forward_sub_rows(const gsparc_frame_layout& L, int64_t Cp);

int launch_preprocess(const gsparc_cloud& cloud, const gsparc_view& view,
                      const gsparc_frame_layout& L, char* frame, cudaStream_t st);
int launch_bin_tiles(const gsparc_frame_layout& L, char* frame, cudaStream_t st,
                     bool dependent = false);
int launch_mlp(const gsparc_cloud& cloud, const double* tx, int B, bool live_only,
               const gsparc_frame_layout& L, char* frame, cudaStream_t st, int stream_ctas = 0);
int launch_raster_forward(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                          double t_eps, int pass, void* img, cudaStream_t st);
int launch_raster_px(const gsparc_frame_layout& L, char* frame, int n_tx, int C, double t_eps,
                     int pass, void* img, cudaStream_t st);
int launch_raster_backward(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                           const void* dL, bool deterministic, cudaStream_t st);
bool raster_bwd_tc_supported(const gsparc_frame_layout& L, int64_t Cp);
int launch_raster_bwd_tc(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                         const void* dL, bool det, cudaStream_t st);
int launch_gauss_backward(const gsparc_cloud& cloud, const gsparc_view& view, const double* tx,
                          int B, const gsparc_frame_layout& L, char* frame, void* grad,
                          int grad_dtype, cudaStream_t st);
int64_t loss_scratch_bytes(int NI, int h, int w, int C);
int launch_loss(const void* img, const void* gt, int dtype, int NI, int h, int w, int C, int sup,
                double lam, void* dimg, double* stats, void* scratch, int64_t scratch_bytes,
                cudaStream_t st);
int launch_adam(double* pos, double* ls, double* rot, double* op, float* mlp, int64_t n, int P,
                const float* g, float* m, float* v, int64_t* step, int* counters,
                const gsparc_adam_config& cfg, cudaStream_t st);

int launch_gt_spectrum(const gsparc_emitter* em_dev, int ne, const double* rx, double wavelength,
                       const double* tx_dev, int B, int w, int h, double scale, int out_dtype,
                       void* out, cudaStream_t st);
int launch_rssi_energy(const void* img, int dtype, int B, int h, int w, int C, const int64_t* sel,
                       int64_t nsel, double* energy, cudaStream_t st);

}  // namespace gs
