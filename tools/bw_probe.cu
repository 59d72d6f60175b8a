// HBM access-pattern probe: what bandwidth does a 6-read/1-write stream reach
// when each CTA walks a strip of width W doubles down y (the sweep's pattern),
// versus a flat grid-stride stream?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 bw_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void flat(const double2 *a, const double2 *b, const double2 *c, const double2 *d,
                     const double2 *e, const double2 *f, double2 *o, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    double2 x = __ldg(a + i), y = __ldg(b + i), z = __ldg(c + i), u = __ldg(d + i), v = __ldg(e + i), w = __ldg(f + i);
    o[i] = make_double2(x.x + y.x + z.x + u.x + v.x + w.x, x.y + y.y + z.y + u.y + v.y + w.y);
  }
}

// CTA = (W/2 lanes-pairs) x L ; strip of W doubles, rows [y0, y0+H), all L layers
template <int W>
__global__ void strip(const double *a, const double *b, const double *c, const double *d, const double *e,
                      const double *f, double *o, int NX, int NY, int L, int H) {
  const int t = threadIdx.x;  // pair within strip
  const int l = threadIdx.y;
  const long x = (long)blockIdx.x * W + 2 * t;
  const int y0 = blockIdx.y * H;
  for (int y = y0; y < y0 + H && y < NY; ++y) {
    const long i = ((long)l * NY + y) * NX + x;
    double2 p = __ldg((const double2 *)(a + i)), q = __ldg((const double2 *)(b + i)),
            r = __ldg((const double2 *)(c + i)), s = __ldg((const double2 *)(d + i)),
            u = __ldg((const double2 *)(e + i)), v = __ldg((const double2 *)(f + i));
    *(double2 *)(o + i) = make_double2(p.x + q.x + r.x + s.x + u.x + v.x, p.y + q.y + r.y + s.y + u.y + v.y);
  }
}

int main() {
  const int L = 4, NY = 1024, NX = 1024;
  const long n = (long)L * NY * NX;
  double *buf[7];
  for (int k = 0; k < 7; ++k) {
    cudaMalloc(&buf[k], n * 8);
    cudaMemset(buf[k], 0, n * 8);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto report = [&](const char *name, float ms, int reps) {
    double gb = 56.0 * n * reps / (ms * 1e-3) / 1e9;
    printf("%-28s %8.1f us/pass  %7.0f GB/s\n", name, ms * 1e3 / reps, gb);
  };
  const int reps = 50;
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    flat<<<blocks, 256>>>((double2 *)buf[0], (double2 *)buf[1], (double2 *)buf[2], (double2 *)buf[3],
                          (double2 *)buf[4], (double2 *)buf[5], (double2 *)buf[6], n / 2);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
      flat<<<blocks, 256>>>((double2 *)buf[0], (double2 *)buf[1], (double2 *)buf[2], (double2 *)buf[3],
                            (double2 *)buf[4], (double2 *)buf[5], (double2 *)buf[6], n / 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    char nm[64];
    snprintf(nm, 64, "flat blocks=%d", blocks);
    report(nm, ms, reps);
  }
#define RUN_STRIP(W)                                                                              \
  for (int H : {8, 32, 128}) {                                                                    \
    dim3 grid(NX / W, NY / H), block(W / 2, L);                                                   \
    strip<W><<<grid, block>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], NX, NY, L, H); \
    cudaEventRecord(e0);                                                                          \
    for (int r = 0; r < reps; ++r)                                                                \
      strip<W><<<grid, block>>>(buf[0], buf[1], buf[2], buf[3], buf[4], buf[5], buf[6], NX, NY, L, H); \
    cudaEventRecord(e1);                                                                          \
    cudaEventSynchronize(e1);                                                                     \
    float ms;                                                                                     \
    cudaEventElapsedTime(&ms, e0, e1);                                                            \
    char nm[64];                                                                                  \
    snprintf(nm, 64, "strip W=%d H=%d", W, H);                                                    \
    report(nm, ms, reps);                                                                         \
  }
  RUN_STRIP(64)
  RUN_STRIP(128)
  RUN_STRIP(256)
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
