// Dependent-chain latency of FP64 add/mul and int add on this GPU (one warp).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, int n) {
  double x = a, y = a;
  int z = (int)a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, 1.0000001);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = __dmul_rn(y, 1.0000001);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) z = z * 3 + 7;
  long long t3 = clock64();
  out[threadIdx.x] = x + y + z;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  const int n = 1 << 16;
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(o, c, 1.0, n);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("per op cycles: dadd %.2f  dmul %.2f  imad+iadd %.2f\n", (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
  }
  return 0;
}
