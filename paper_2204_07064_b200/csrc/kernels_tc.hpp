// kernels_tc.hpp — tcgen05/TMEM/TMA dense cached-conv (see kernels_tc.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "common.hpp"

namespace scb {

struct TcParams {
  // tiling
  int BN;               // 32 | 64 | 128 | 256
  int R, G;             // tile = G streams x R rows (R*G <= 128)
  int tiles_per_stream; // when G == 1
  int m_tiles;
  int n_kblocks;        // taps_view * cblocks
  int cblocks;          // 32-channel blocks per tap (view channels padded to 32)
  // A (input window) coordinates in the tensor-map view (channel, row, stream)
  int a_c0;             // channel offset of the view
  int a_row0;           // first window row of output row 0
  int a_tap_rows;       // rows between taps
  int win;              // 1: fp32 narrow tile, A box = 128 + halo rows per 32-channel block
  int halo;             // (taps - 1) * a_tap_rows
  int wres;             // 1 (win only): the whole weight (hi + lo) is resident in shared memory
  // epilogue (same meaning as ConvParams)
  int pre_act;
  float pre_alpha;
  int post_act;
  float post_alpha;
  int gate;
  int nout;
  int t_out;
  int streams;
  const float* bias;
  float* out;
  int64_t out_sstride;
  int64_t out_base;
  int out_rstride;
  const float* res;
  int64_t res_sstride;
  int res_fstride;
  int res_off;
  int res_f0;
  int res_act;
  float res_alpha;
  int bf16;   // 1: bf16 operands (kind::f16), fp32 accumulate; 0: fp32-accurate (3xTF32 or 3xFP16)
  int f16;    // fp32 plans: 1 = 3xFP16 (fp16 hi / lo, per-row power-of-two scaling), 0 = 3xTF32
  int f16_sw; // 3xFP16: the layer's weight scale exponent (weights were multiplied by 2^f16_sw)
  int awin;    // 3xFP16 non-window tiles: one A load per 32-channel block serves every tap (box
               // of G streams x (R + halo) rows <= 192), else one A box per K-slab
  int a_bf, r_bf, o_bf;  // bf16 plans: input / residual / output buffer holds bf16 (else fp32)
  int cbmaj;  // 1: K-slabs channel-block major (layers that may run in window mode), else tap major
  // chained 1x1 conv (fp32, BN = 128, one N tile): the drain turns the first conv's tile
  // h = act2(act1(acc + bias)) into the A operand of a second GEMM (chain K-slabs of 32
  // channels, weights at K offset n_kblocks x 32 of the same weight map) whose tile goes
  // through the epilogue above (bias2, post act, residual, output of the second conv).
  int chain;            // 0: single conv; else K-slabs of the second conv (cin2 / 32)
  const float* bias2;   // second conv's bias (nout)
  int chain_one;
  int mid_bf;           // bf16 plans: the two-launch form stores the intermediate as bf16
  int ck;               // fp32 BN = 128: K-slabs per TMEM chunk accumulator (1, 2, 4)        // 1: the chained GEMM accumulates its K-slabs in one TMEM chunk
  int mid_act1, mid_act2;
  float mid_alpha1, mid_alpha2;
  int debug;  // experiments only (SC_TC_DEBUG): 2 no correction MMAs (timing only), 4 no residual L2 prefetch, 32 trace (SC_TC_TRACE_OP)
};

// map_out: output rows (dims out_rstride x t_out x streams, base at the first output row),
// map_res: residual rows (dims res_fstride x t_out x streams, base at res_f0); box 32 x R x G.
void launch_conv_tc(const CUtensorMap& map_a, const CUtensorMap& map_w, const CUtensorMap& map_out,
                    const CUtensorMap& map_res, const TcParams& p, cudaStream_t st);

void tc_trace_dump(long long* host);  // experiments: SC_TC_DEBUG & 32 timestamps

}  // namespace scb
