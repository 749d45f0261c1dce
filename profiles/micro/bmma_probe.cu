#include <cstdint>
#include <cstdio>
__global__ void k(const uint32_t* a, const uint32_t* b, int* out, int iters) {
  uint32_t A0 = a[threadIdx.x], A1 = a[threadIdx.x + 32], A2 = a[threadIdx.x + 64], A3 = a[threadIdx.x + 96];
  uint32_t B0 = b[threadIdx.x], B1 = b[threadIdx.x + 32];
  int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c0), "+r"(c1), "+r"(c2), "+r"(c3)
                 : "r"(A0), "r"(A1), "r"(A2), "r"(A3), "r"(B0), "r"(B1));
    B0 += i; 
  }
  out[threadIdx.x + blockIdx.x * 32] = c0 ^ c1 ^ c2 ^ c3;
}
int main() { return 0; }
