// Launchers of the specialized general-map kernels (hxg_gen_*.cu).
// Each returns 0 on success, 1 if no specialization exists for p, <0 on error.
#pragma once
#include <cuda_runtime.h>

namespace hxg {
struct V2Args;
struct AffV2Args;
struct ExtArgs;
int launch_v2_H1(int p, const V2Args &a, cudaStream_t st);
int launch_v2_hcurl(int p, const V2Args &a, cudaStream_t st);
int launch_v2_hdiv(int p, const V2Args &a, cudaStream_t st);
int launch_v2_l2(int p, const V2Args &a, cudaStream_t st);
int launch_aff_H1(int p, const AffV2Args &a, cudaStream_t st);
int launch_aff_hcurl(int p, const AffV2Args &a, cudaStream_t st);
int launch_aff_hdiv(int p, const AffV2Args &a, cudaStream_t st);
int launch_aff_l2(int p, const AffV2Args &a, cudaStream_t st);
int launch_ext_H1(int p, const ExtArgs &a, cudaStream_t st);
int launch_ext_hcurl(int p, const ExtArgs &a, cudaStream_t st);
int launch_ext_hdiv(int p, const ExtArgs &a, cudaStream_t st);
int launch_ext_l2(int p, const ExtArgs &a, cudaStream_t st);
// specialized metric kernel (hxg_metric.cuh), rule sizes L = 2..11; returns 1 if none
// exists for L.  It writes every element's status word (no memset before it).
struct MetArgs {
    int E;
    const int *kind;
    const double *params, *coef, *wgrid, *tables;
    double *metric;
    int *status;
    int status_or;  // 1: OR bit 0 into the (pre-zeroed / pre-flagged) word, 0: write it whole
};
int launch_met_H1(int L, const MetArgs &a, cudaStream_t st);
int launch_met_hcurl(int L, const MetArgs &a, cudaStream_t st);
int launch_met_hdiv(int L, const MetArgs &a, cudaStream_t st);
int launch_met_l2(int L, const MetArgs &a, cudaStream_t st);
}  // namespace hxg
