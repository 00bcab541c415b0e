// Read-stream ceiling of this B200: persistent CTAs stream 32 GiB through a TMA
// bulk-copy ring (one producer lane, 7 consumer warps), no compute.  The LSQR
// pass (K4) is compared against it in DESIGN.md section 4.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/bw_read_ceiling.cu -o bw && ./bw
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned su32(const void* p){return (unsigned)__cvta_generic_to_shared(p);}
__device__ __forceinline__ void minit(uint64_t* b, unsigned c){asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"::"r"(su32(b)),"r"(c):"memory");}
__device__ __forceinline__ void mexp(uint64_t* b, unsigned x){asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(su32(b)),"r"(x):"memory");}
__device__ __forceinline__ void marr(uint64_t* b){asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"::"r"(su32(b)):"memory");}
__device__ __forceinline__ void mwait(uint64_t* b, unsigned ph){unsigned ok=0; do{asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}":"=r"(ok):"r"(su32(b)),"r"(ph):"memory");}while(!ok);}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned n, uint64_t* b, uint64_t pol){asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"::"r"(su32(d)),"l"(s),"r"(n),"r"(su32(b)),"l"(pol):"memory");}
__global__ void __launch_bounds__(256,1) k(const char* A, size_t bytes, int tile, int S, double* out) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full=(uint64_t*)(sm + (size_t)S*tile); uint64_t* empty=full+S;
  int tid=threadIdx.x, warp=tid>>5, lane=tid&31;
  size_t nt=bytes/tile, t0=blockIdx.x*nt/gridDim.x, t1=(blockIdx.x+1)*nt/gridDim.x, n=t1-t0;
  if(tid==0){for(int s=0;s<S;++s){minit(&full[s],1);minit(&empty[s],7);} asm volatile("fence.mbarrier_init.release.cluster;");}
  __syncthreads();
  double acc=0;
  if(warp==7){ if(lane==0){ uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;":"=l"(pol));
      for(size_t i=0;i<n;++i){int s=i%S; if(i>=S) mwait(&empty[s],((i/S)-1)&1); mexp(&full[s],tile); bulk(sm+(size_t)s*tile, A+(t0+i)*(size_t)tile, tile, &full[s], pol);} } }
  else { for(size_t i=0;i<n;++i){int s=i%S; mwait(&full[s],(i/S)&1); const double* t=(const double*)(sm+(size_t)s*tile); acc+=t[warp*32+lane]; __syncwarp(); if(lane==0) marr(&empty[s]);} }
  if(acc==12345.0) out[0]=acc;
}
int main(){ size_t bytes=32ull<<30; char* A; cudaMalloc(&A,bytes); cudaMemset(A,0,bytes); double* o; cudaMalloc(&o,8);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int cfgs[][2]={{65536,3},{32768,6},{49152,4},{16384,12},{98304,2}};
  for(auto& c: cfgs){ int tile=c[0],S=c[1]; size_t smem=(size_t)S*tile+256; cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)smem);
    for(int r=0;r<3;++r){ cudaEventRecord(e0); k<<<148,256,smem>>>(A,bytes,tile,S,o); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(r==2) printf("tile %d S %d: %.3f ms %.0f GB/s\n",tile,S,ms,bytes/ms/1e6);} }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
