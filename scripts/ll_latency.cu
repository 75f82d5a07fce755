// Inter-CTA handshake latency on the B200 (measurement tooling for the C2
// resident solve): G CTAs in a ring, one per SM; in round s every
// CTA publishes tag s to its own mailbox and waits for tag s in both
// neighbours' mailboxes.  The time per round is the per-hop latency of the
// sweep-to-sweep chain that k_resident's LL mailbox pays every sweep.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ll_latency scripts/ll_latency.cu
//   /tmp/ll_latency
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rel(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st4(unsigned long long* p, unsigned long long a, unsigned long long b,
                                    unsigned long long c, unsigned long long d) {
  asm volatile("st.relaxed.gpu.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
               : "memory");
}
__device__ __forceinline__ void ld4(const unsigned long long* p, unsigned long long (&v)[4]) {
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ void ld2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// mode 0: thread 0 of each CTA publishes a flag and polls the two neighbour flags
// mode 1: every thread publishes 4 16-B LL entries and polls 4 of the neighbours'
// mode 2: mode 1 + __syncthreads per round (k_resident's sweep without compute)
// mode 3: mode 0 + __syncthreads per round (thread 0 polls, the CTA waits at the barrier)
// mode 4: mode 1 with the mailbox slot alternating by round parity (k_resident's two slots)
// mode 5: k_resident's exchange: 2 slots, one column pair per thread (nx/2 = 512 pairs), the four
//         entries polled together, __nanosleep(100) between polls, barrier
// mode 6: mode 5 without the back-off
// mode 8: mode 5 with each pair's two entries as ONE 32-B access (v4.u64, sm_100)
// mode 9: plain 16-B data per pair (no tags) + one flag per warp and row: the lanes store, __syncwarp,
//         lane 0 st.release.gpu of the round; the reader's lane 0 polls the flag (ld.acquire.gpu),
//         __syncwarp, then every lane loads its pair (ld.relaxed.gpu)
// mode 7: mode 5 with the pair's two entries in separate halves of the row (entries q and
//         np + q): every warp-wide access covers whole 32-B sectors
__global__ void k_ring(unsigned long long* mb, int rounds, int mode, int nx, long long* cycles) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int up = c > 0 ? c - 1 : G - 1, dn = c < G - 1 ? c + 1 : 0;
  grid.sync();
  const long long t0 = clock64();
  for (int s = 1; s <= rounds; ++s) {
    const unsigned long long tag = (unsigned long long)s << 32;
    if (mode == 0 || mode == 3) {
      if (tid == 0) {
        st_rel(mb + (size_t)c * 16, tag);
        while (ld_rel(mb + (size_t)up * 16) < tag) {
        }
        while (ld_rel(mb + (size_t)dn * 16) < tag) {
        }
      }
      if (mode == 3) __syncthreads();
    } else if (mode == 9) {
      const int slot = s & 1;
      const int np = nx / 2, lane = tid & 31, warp = tid >> 5;
      // data [slot][cta][2 rows][np pairs][2]; flags [slot][cta][2 rows][np / 32 warps] (128-B apart)
      unsigned long long* data = mb + (size_t)slot * G * 2 * 2 * np;
      unsigned long long* flg = mb + (size_t)2 * G * 2 * 2 * np + (size_t)slot * G * 2 * (np / 32) * 16;
      for (int q = tid; q < np; q += nt) {
        st2(data + ((size_t)c * 2 + 0) * 2 * np + 2 * q, tag | 1, tag | 2);
        st2(data + ((size_t)c * 2 + 1) * 2 * np + 2 * q, tag | 1, tag | 2);
        __syncwarp();
        if (lane == 0) {
          const int wq = q >> 5;
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flg + (((size_t)c * 2 + 0) * (np / 32) + wq) * 16),
                       "l"((unsigned long long)s) : "memory");
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flg + (((size_t)c * 2 + 1) * (np / 32) + wq) * 16),
                       "l"((unsigned long long)s) : "memory");
        }
      }
      for (int q = tid; q < np; q += nt) {
        const int wq = q >> 5;
        if (lane == 0) {
          const unsigned long long* fu = flg + (((size_t)up * 2 + 1) * (np / 32) + wq) * 16;
          const unsigned long long* fd = flg + (((size_t)dn * 2 + 0) * (np / 32) + wq) * 16;
          unsigned long long a, b;
          do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(fu) : "memory");
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(b) : "l"(fd) : "memory");
          } while (a != (unsigned long long)s || b != (unsigned long long)s);
        }
        __syncwarp();
        unsigned long long a0, b0, a1, b1;
        ld2(data + ((size_t)up * 2 + 1) * 2 * np + 2 * q, a0, b0);
        ld2(data + ((size_t)dn * 2 + 0) * 2 * np + 2 * q, a1, b1);
        if ((a0 >> 32) != (unsigned long long)s || (a1 >> 32) != (unsigned long long)s) asm volatile("trap;");
      }
      __syncthreads();
    } else if (mode == 8) {
      const int slot = s & 1;
      const int np = nx / 2;
      unsigned long long* base = mb + (size_t)slot * G * 8 * np;
      for (int q = tid; q < np; q += nt) {
        st4(base + ((size_t)c * 2 + 0) * 4 * np + 4 * q, tag | 1, tag | 2, tag | 3, tag | 4);
        st4(base + ((size_t)c * 2 + 1) * 4 * np + 4 * q, tag | 1, tag | 2, tag | 3, tag | 4);
      }
      const unsigned long long w = (unsigned long long)s;
      for (int q = tid; q < np; q += nt) {
        const unsigned long long* e0 = base + ((size_t)up * 2 + 1) * 4 * np + 4 * q;
        const unsigned long long* e1 = base + ((size_t)dn * 2 + 0) * 4 * np + 4 * q;
        unsigned long long a[4], b[4];
        ld4(e0, a);
        ld4(e1, b);
        auto bad = [&](const unsigned long long(&v)[4]) {
          return (v[0] >> 32) != w || (v[1] >> 32) != w || (v[2] >> 32) != w || (v[3] >> 32) != w;
        };
        while (bad(a) || bad(b)) {
          if (bad(a)) ld4(e0, a);
          if (bad(b)) ld4(e1, b);
        }
      }
      __syncthreads();
    } else if (mode >= 5) {
      const int slot = s & 1;
      const int np = nx / 2;
      unsigned long long* base = mb + (size_t)slot * G * 8 * np;  // [slot][cta][2 rows][2 np entries][2]
      for (int q = tid; q < np; q += nt) {
        const int o0 = mode == 7 ? 2 * q : 4 * q, o1 = mode == 7 ? 2 * (np + q) : 4 * q + 2;
        unsigned long long* f = base + ((size_t)c * 2 + 0) * 4 * np;
        unsigned long long* l = base + ((size_t)c * 2 + 1) * 4 * np;
        st2(f + o0, tag | 1, tag | 2);
        st2(f + o1, tag | 3, tag | 4);
        st2(l + o0, tag | 1, tag | 2);
        st2(l + o1, tag | 3, tag | 4);
      }
      const unsigned long long w = (unsigned long long)s;
      for (int q = tid; q < np; q += nt) {
        const int o0 = mode == 7 ? 2 * q : 4 * q, o1 = mode == 7 ? 2 * (np + q) : 4 * q + 2;
        const unsigned long long* e[4] = {base + ((size_t)up * 2 + 1) * 4 * np + o0,
                                          base + ((size_t)up * 2 + 1) * 4 * np + o1,
                                          base + ((size_t)dn * 2 + 0) * 4 * np + o0,
                                          base + ((size_t)dn * 2 + 0) * 4 * np + o1};
        unsigned long long a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) ld2(e[i], a[i], b[i]);
        for (;;) {
          bool ok = true;
#pragma unroll
          for (int i = 0; i < 4; ++i) ok = ok && (a[i] >> 32) == w && (b[i] >> 32) == w;
          if (ok) break;
          if (mode == 5) __nanosleep(100);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if ((a[i] >> 32) != w || (b[i] >> 32) != w) ld2(e[i], a[i], b[i]);
        }
      }
      __syncthreads();
    } else {
      const int slot = mode == 4 ? (s & 1) : 0;
      unsigned long long* base = mb + (size_t)slot * G * 4 * nx;  // [slot][cta][2 rows][nx][2]
      for (int q = tid; q < nx; q += nt) {
        st2(base + ((size_t)c * 2 + 0) * 2 * nx + 2 * q, tag | q, tag | 1);
        st2(base + ((size_t)c * 2 + 1) * 2 * nx + 2 * q, tag | q, tag | 2);
      }
      for (int q = tid; q < nx; q += nt) {
        const unsigned long long* e0 = base + ((size_t)up * 2 + 1) * 2 * nx + 2 * q;
        const unsigned long long* e1 = base + ((size_t)dn * 2 + 0) * 2 * nx + 2 * q;
        unsigned long long a0, b0, a1, b1;
        ld2(e0, a0, b0);
        ld2(e1, a1, b1);
        // one slot: a neighbour may already have published round s+1 (tags
        // compare >=); two slots: exactly round s (as k_resident)
        const unsigned long long w = (unsigned long long)s;
        auto bad = [&](unsigned long long a, unsigned long long b) {
          return mode == 4 ? ((a >> 32) != w || (b >> 32) != w) : ((a >> 32) < w || (b >> 32) < w);
        };
        while (bad(a0, b0) || bad(a1, b1)) {
          if (bad(a0, b0)) ld2(e0, a0, b0);
          if (bad(a1, b1)) ld2(e1, a1, b1);
        }
      }
      if (mode >= 2) __syncthreads();
    }
  }
  const long long t1 = clock64();
  if (tid == 0) cycles[c] = t1 - t0;
}

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int nx = 1024, rounds = 2000;
  unsigned long long* mb;
  long long* cyc;
  cudaMalloc(&mb, (size_t)4 * nsm * 8 * nx * 8 + 4096);
  cudaMalloc(&cyc, nsm * sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"flag, 1 thread", "LL 512 thr", "LL 512 thr + bar", "flag + bar", "LL 2 slots", "k_resident exchange", "k_resident exchange, no back-off",
                         "k_resident exchange, sector-contiguous entries", "k_resident exchange, 32-B pair entries",
                         "plain pairs + per-warp release/acquire flag"};
  // payload sweep of the 32-B pair entries (mode 8): columns per row
  for (int cols : {1024, 512, 256, 64}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(mb, 0, (size_t)4 * nsm * 8 * nx * 8 + 4096);
      int r = rounds, m = 8, n = cols;
      void* args[] = {&mb, &r, &m, &n, &cyc};
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)k_ring, nsm, 512, args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"mode\": \"32-B pair entries\", \"cols\": %d, \"us_per_round\": %.3f}\n", cols, 1000.0 * ms / rounds);
    }
  }
  for (int threads : {512, 256}) {
    for (int mode = 0; mode < 10; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(mb, 0, (size_t)4 * nsm * 8 * nx * 8 + 4096);
        int r = rounds, m = mode, n = nx;
        void* args[] = {&mb, &r, &m, &n, &cyc};
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchCooperativeKernel((void*)k_ring, nsm, threads, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
          printf("launch failed: %s\n", cudaGetErrorString(err));
          return 1;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h[1024];
        cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("{\"mode\": \"%s\", \"threads\": %d, \"ctas\": %d, \"us_per_round\": %.3f, \"cycles_per_round\": %.0f}\n",
               names[mode], threads, nsm, 1000.0 * ms / rounds, (double)mx / rounds);
      }
    }
  }
  (void)clk;
  return 0;
}
