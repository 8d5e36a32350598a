// Device probe: properties, fp64 FMA throughput, fp64 streaming bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
__global__ void dfma_kernel(double* out, int iters, double a, double b){
  double x0=threadIdx.x*1e-3, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int k=0;k<16;k++){ x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
      x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);}
  }
  double s=x0+x1+x2+x3+x4+x5+x6+x7; if(s==123.456) out[0]=s;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("name=%s sms=%d cc=%d.%d l2=%d smem/blk optin=%zu smem/sm=%zu regs/sm=%d clock_khz=%d memclk_khz=%d busw=%d\n",
    p.name,p.multiProcessorCount,p.major,p.minor,p.l2CacheSize,p.sharedMemPerBlockOptin,p.sharedMemPerMultiprocessor,p.regsPerMultiprocessor,p.clockRate,p.memoryClockRate,p.memoryBusWidth);
  double* d; CK(cudaMalloc(&d,8));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=4096; int blocks=p.multiProcessorCount*8, threads=256;
  dfma_kernel<<<blocks,threads>>>(d,16,1.0000001,1e-9); CK(cudaDeviceSynchronize());
  for(int rep=0;rep<3;rep++){
  cudaEventRecord(e0); dfma_kernel<<<blocks,threads>>>(d,iters,0.9999999,1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  double fmas=(double)blocks*threads*iters*16*8;
  printf("dfma: %.3f ms  %.2f TFMA/s = %.2f TFLOP/s (fp64)\n",ms,fmas/ms/1e9,2*fmas/ms/1e9);
  }
  size_t n=(size_t)1<<27; // 2^27 double2 = 2 GiB
  double2 *a,*b; CK(cudaMalloc(&a,n*16)); CK(cudaMalloc(&b,n*16)); cudaMemset(a,0,n*16);
  for(int rep=0;rep<4;rep++){
  cudaEventRecord(e0); copy_kernel<<<p.multiProcessorCount*16,512>>>(a,b,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  printf("copy fp64 2x2GiB: %.3f ms  %.1f GB/s\n",ms,2.0*n*16/ms/1e6);
  }
  return 0;
}
