// Debug harness: run general_v3_kernel<H1, 7, 8> on one element with a synthetic metric
// and dump stage-A / stage-B intermediates of unit (b=0,a=0,j3=0,i3=0), j2 = 0.

#include "../paper_1711_00984_b200/csrc/hxg_general_v3.cuh"
#include "../paper_1711_00984_b200/csrc/hxg_kernels.cuh"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace hxg;
int main() {
  constexpr int S = H1, P = 7, L = 8;
  using C = V3Cfg<S, P, L>;
  double *tab; cudaMalloc(&tab, TAB_TOTAL * 8);
  tables_kernel<<<1, 128>>>(L, nullptr, nullptr, tab);
  std::vector<double> htab(TAB_TOTAL); cudaMemcpy(htab.data(), tab, TAB_TOTAL*8, cudaMemcpyDeviceToHost);
  const int L3 = L*L*L, NF = C::NF;
  std::vector<double> met(NF * L3);
  for (int i = 0; i < NF * L3; ++i) met[i] = std::sin(0.37 * i) + 0.1 * (i % 7);
  double *dmet; cudaMalloc(&dmet, met.size()*8); cudaMemcpy(dmet, met.data(), met.size()*8, cudaMemcpyHostToDevice);
  long long Pk = (long long)C::N * (C::N + 1) / 2;
  double *out; cudaMalloc(&out, Pk * 8);
  double *dbg; cudaMalloc(&dbg, 4096*8); cudaMemset(dbg, 0, 4096*8);
#if 1
  cudaMemcpyToSymbol(hxg_dbg, &dbg, sizeof(double*));
#endif
  V3Args a{tab, dmet, out, Pk, 1, 1};
  auto k = general_v3_kernel<S, P, L>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  k<<<1, V3_THREADS, C::SMEM_BYTES>>>(a);
  cudaError_t e = cudaDeviceSynchronize(); printf("err %s\n", cudaGetErrorString(e));
  std::vector<double> h(4096); cudaMemcpy(h.data(), dbg, 4096*8, cudaMemcpyDeviceToHost);
  // CPU: T(f,k,l) = htab[TAB_T + (f*KT + k)*LT + l]
  auto T = [&](int f, int kk, int l) { return htab[TAB_T + (f*KT + kk)*LT + l]; };
  constexpr CPair pp = make_pair_plan(S, 0, 0);
  double maxA = 0, maxB = 0;
  std::vector<double> Ab(pp.ng*64, 0.0);
  for (int g = 0; g < pp.ng; ++g) for (int l = 0; l < L; ++l) for (int m = 0; m < L; ++m) {
    double acc = 0;
    for (int t = 0; t < pp.nt; ++t) { if (pp.t_g[t] != g) continue; double s = 0;
      for (int n = 0; n < L; ++n) s += met[pp.t_field[t]*L3 + n*L*L + l*L + m] * T(pp.t_fr[t], 0, n) * T(pp.t_fs[t], 0, n);
      acc += pp.t_sign[t] * s; }
    Ab[(g*8 + m)*8 + l] = acc;
    maxA = fmax(maxA, fabs(acc - h[(g*8+m)*8+l]));
  }
  std::vector<double> Bcpu(pp.nh*64, 0.0);
  for (int hh = 0; hh < pp.nh; ++hh) for (int i2 = 0; i2 < 8; ++i2) for (int l = 0; l < L; ++l) {
    double acc = 0;
    for (int g = 0; g < pp.ng; ++g) { if (pp.g_h[g] != hh) continue;
      for (int m = 0; m < L; ++m) acc += T(pp.g_fr[g], i2, m) * T(pp.g_fs[g], 7, m) * Ab[(g*8+m)*8+l]; }
    Bcpu[(hh*8 + i2)*8 + l] = acc;
    double gv = h[1024 + (hh*8 + i2)*8 + l];
    if (fabs(acc - gv) > maxB) maxB = fabs(acc - gv);
    if (hh == 0 && l < 3) printf("h0 i2=%d l=%d cpu %.6f gpu %.6f\n", i2, l, acc, gv);
  }
  printf("max |dA| %.3e  max |dB| %.3e  ng %d nh %d\n", maxA, maxB, pp.ng, pp.nh);
  for (int ln = 0; ln < 8; ++ln) printf("lane %d Ta0 %.4f Ta1 %.4f Tb0 %.4f\n", ln*4, h[2048+ln*4], h[2080+ln*4], h[2112+ln*4]);
  std::vector<double> ho(Pk); cudaMemcpy(ho.data(), out, Pk*8, cudaMemcpyDeviceToHost);
  // row J = 0 (j1=j2=j3=0), columns i3=0 block: I = i1 + 8*i2
  double maxC = 0;
  for (int i2 = 0; i2 < 8; ++i2) { for (int i1 = 0; i1 < 8; ++i1) {
    double acc = 0;
    for (int hh = 0; hh < pp.nh; ++hh) for (int l = 0; l < L; ++l)
      acc += T(pp.h_fs[hh], 0, l) * T(pp.h_fr[hh], i1, l) * Bcpu[(hh*8 + i2)*8 + l];
    double gv = ho[i1 + 8*i2];
    maxC = fmax(maxC, fabs(acc - gv));
    if (i2 < 2) printf("i2=%d i1=%d cpu %.5f gpu %.5f\n", i2, i1, acc, gv);
  } }
  printf("max |dC| %.3e\n", maxC);
  printf("YF %d\n", (int)V2Cfg<S,P,L>::yform(0,0));
  // registers: expected per lane
  int badreg = 0;
  for (int ln = 0; ln < 32; ++ln) { int g8 = ln >> 2, t4 = ln & 3;
    for (int ks = 0; ks < 4; ++ks) { int k = ks*4 + t4; int r = k / L, l = k % L;
      double R0e = T(pp.r_code[r], g8, l);
      double gR0 = h[2048 + ks*32 + ln];
      int hl[2], nq = 0; for (int hh = 0; hh < pp.nh; ++hh) if (pp.h_r[hh] == r) hl[nq++] = hh;
      double Yc0 = T(pp.h_fs[hl[0]], g8, l), Yc1 = T(pp.h_fs[hl[1]], g8, l);
      int Ro0 = hl[0]*64 + l, Ro1 = hl[1]*64 + l;
      if (fabs(R0e - gR0) > 1e-14 || fabs(Yc0 - h[2304+ks*32+ln]) > 1e-14 || fabs(Yc1 - h[2560+ks*32+ln]) > 1e-14 || Ro0 != (int)h[2816+ks*32+ln] || Ro1 != (int)h[3072+ks*32+ln]) {
        if (badreg < 10) printf("lane %d ks %d: R0 %g/%g Yc0 %g/%g Yc1 %g/%g Ro0 %d/%d Ro1 %d/%d\n", ln, ks, R0e, gR0, Yc0, h[2304+ks*32+ln], Yc1, h[2560+ks*32+ln], Ro0, (int)h[2816+ks*32+ln], Ro1, (int)h[3072+ks*32+ln]);
        badreg++; } } }
  printf("bad regs %d\n", badreg);
  // staging row 0 of last j2 (=7): expected from Bcpu (j2 = 7)
  double maxS = 0; int SWv = C::SW;
  for (int i2 = 0; i2 < 8; ++i2) for (int i1 = 0; i1 < 8; ++i1) {
    double acc = 0;
    for (int hh = 0; hh < pp.nh; ++hh) for (int l = 0; l < L; ++l)
      acc += T(pp.h_fs[hh], 0, l) * T(pp.h_fr[hh], i1, l) * Bcpu[(hh*8 + i2)*8 + l];
    double g0 = h[3328 + i2*8 + i1], g1 = h[3328 + 1 + i2*8 + i1];
    double dd = fmin(fabs(acc - g0), fabs(acc - g1)); maxS = fmax(maxS, dd);
    if (i2 == 1 && i1 < 3) printf("stage row0 i2=1 i1=%d cpu %.5f gpu(pad0) %.5f gpu(pad1) %.5f\n", i1, acc, g0, g1);
  }
  printf("max |dS| %.3e\n", maxS);
  return 0;
}
