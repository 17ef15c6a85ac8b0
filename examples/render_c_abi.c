/* A plain-C client of the C ABI (include/p2s.h): no PyTorch, no C++. Builds a handle whose basis
 * is one centred delta per function scaled so that sum_k beta_k phi_k is the identity PSF
 * (K = 4, S = 5, beta_k = 1/K from b3 with zero weights), renders a 3-channel 67 x 150 ramp
 * with a uniform tilt of (1, 0) pixels, and checks the closed form out(y, x) = I(y, max(x - 1, 0))
 * (PAPER.md:172 / SURVEY P4: an integer shift moves content right by one pixel, column 0
 * replicated) within the fp16 operand rounding. Then the adjoint: dL/dt of L = sum(out) and
 * p2s_mlp_backward's dL/dz (zero here: the weights are zero). Exit status 0 = pass.
 *   gcc -O2 -Iinclude -I$CUDA/include examples/render_c_abi.c -Lpaper_2107_11627_b200 -lp2s
 *       -L$CUDA/lib64 -lcudart -Wl,-rpath,... -o render_c_abi */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "p2s.h"

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                   \
      return 2;                                                                  \
    }                                                                            \
  } while (0)
#define PK(x)                                                                    \
  do {                                                                           \
    p2s_status s_ = (x);                                                         \
    if (s_ != P2S_OK) {                                                          \
      fprintf(stderr, "%s: %s %s\n", #x, p2s_status_string(s_), p2s_last_cuda_error()); \
      return 3;                                                                  \
    }                                                                            \
  } while (0)

int main(void) {
  enum { K = 4, S = 5, NIN = 33, H1 = 16, H2 = 16, B = 1, C = 3, H = 67, W = 150 };
  static float taps[K * S * S], W1[H1 * NIN], b1[H1], W2[H2 * H1], b2[H2], W3[K * H2], b3[K];
  for (int k = 0; k < K; ++k) {
    taps[k * S * S + (S / 2) * S + S / 2] = 1.f;  /* centred delta */
    b3[k] = 1.f / K;                               /* beta_k = 1/K everywhere */
  }
  p2s_basis basis = {K, S, taps};
  p2s_mlp mlp = {NIN, H1, H2, K, W1, b1, W2, b2, W3, b3};
  p2s_handle* h = NULL;
  PK(p2s_init(&basis, &mlp, &h));

  const size_t npx = (size_t)H * W;
  float* img = malloc(sizeof(float) * C * npx);
  float* out = malloc(sizeof(float) * C * npx);
  float* tilt = malloc(sizeof(float) * 2 * npx);
  for (int c = 0; c < C; ++c)
    for (size_t i = 0; i < npx; ++i) img[c * npx + i] = (float)((i % W) + 3 * (i / W) + 7 * c) / (W + 3 * H + 21);
  for (size_t i = 0; i < npx; ++i) { tilt[i] = 1.f; tilt[npx + i] = 0.f; }
  float *d_img, *d_z, *d_t, *d_out, *d_g, *d_gb, *d_gt, *d_gz;
  CK(cudaMalloc((void**)&d_img, sizeof(float) * C * npx));
  CK(cudaMalloc((void**)&d_z, sizeof(float) * NIN * npx));
  CK(cudaMalloc((void**)&d_t, sizeof(float) * 2 * npx));
  CK(cudaMalloc((void**)&d_out, sizeof(float) * C * npx));
  CK(cudaMalloc((void**)&d_g, sizeof(float) * C * npx));
  CK(cudaMalloc((void**)&d_gb, sizeof(float) * K * npx));
  CK(cudaMalloc((void**)&d_gt, sizeof(float) * 2 * npx));
  CK(cudaMalloc((void**)&d_gz, sizeof(float) * NIN * npx));
  CK(cudaMemcpy(d_img, img, sizeof(float) * C * npx, cudaMemcpyHostToDevice));
  CK(cudaMemset(d_z, 0, sizeof(float) * NIN * npx));
  CK(cudaMemcpy(d_t, tilt, sizeof(float) * 2 * npx, cudaMemcpyHostToDevice));
  p2s_image im = {d_img, B, C, H, W};
  PK(p2s_render(h, im, d_z, d_t, d_out, NULL));
  CK(cudaMemcpy(out, d_out, sizeof(float) * C * npx, cudaMemcpyDeviceToHost));
  double err = 0;
  for (int c = 0; c < C; ++c)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const double ref = img[c * npx + (size_t)y * W + (x > 0 ? x - 1 : 0)];
        err = fmax(err, fabs(out[c * npx + (size_t)y * W + x] - ref));
      }
  printf("render (delta basis, shift by one column): max |out - closed form| = %.3e\n", err);
  /* adjoint of L = sum(out): dL/dout = 1 */
  for (size_t i = 0; i < C * npx; ++i) out[i] = 1.f;
  CK(cudaMemcpy(d_g, out, sizeof(float) * C * npx, cudaMemcpyHostToDevice));
  PK(p2s_backward(h, im, d_z, d_t, d_g, d_gb, d_gt, NULL, NULL));
  PK(p2s_mlp_backward(h, d_z, d_gb, B, H, W, d_gz, NULL));
  float* gz = malloc(sizeof(float) * NIN * npx);
  CK(cudaMemcpy(gz, d_gz, sizeof(float) * NIN * npx, cudaMemcpyDeviceToHost));
  double gzmax = 0;
  for (size_t i = 0; i < NIN * npx; ++i) gzmax = fmax(gzmax, fabs(gz[i]));
  printf("adjoint: max |dL/dz| = %.3e (zero weights)\n", gzmax);
  p2s_destroy(h);
  cudaFree(d_img); cudaFree(d_z); cudaFree(d_t); cudaFree(d_out); cudaFree(d_g); cudaFree(d_gb); cudaFree(d_gt);
  cudaFree(d_gz);
  free(img); free(out); free(tilt); free(gz);
  const int ok = err <= 2e-3 && gzmax == 0.0;
  printf("%s\n", ok ? "render_c_abi: ok" : "render_c_abi: FAILED");
  return ok ? 0 : 1;
}
