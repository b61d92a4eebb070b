// Microbenchmarks for the roofline denominators the driver does not measure:
// write-only and read-only HBM bandwidth (fp64 128-bit vectors), and the FP64 FMA rate.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);exit(1);}}while(0)

__global__ void wr(double2* __restrict__ p, size_t n2, double v){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x*blockDim.x;
  for(; i<n2; i+=st) p[i] = make_double2(v, v+1.0);
}
__global__ void wr_cs(double2* __restrict__ p, size_t n2, double v){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x*blockDim.x;
  for(; i<n2; i+=st) __stcs(p+i, make_double2(v, v+1.0));
}
__global__ void rd(const double2* __restrict__ p, size_t n2, double* out){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x*blockDim.x;
  double a=0,b=0;
  #pragma unroll 8
  for(; i<n2; i+=st){ double2 x = __ldcs(p+i); a+=x.x; b+=x.y; }
  if(a+b==12345.678) out[0]=a;
}
__global__ void dfma(double* out, int iters){
  double a=threadIdx.x*1e-3, b=1.0000001, c0=0.1,c1=0.2,c2=0.3,c3=0.4,c4=.5,c5=.6,c6=.7,c7=.8;
  for(int k=0;k<iters;k++){ c0=fma(c0,b,a);c1=fma(c1,b,a);c2=fma(c2,b,a);c3=fma(c3,b,a);c4=fma(c4,b,a);c5=fma(c5,b,a);c6=fma(c6,b,a);c7=fma(c7,b,a);}
  double s=c0+c1+c2+c3+c4+c5+c6+c7; if(s==1.2345) out[0]=s;
}
__global__ void ex2f(float* out, int iters){
  float a=threadIdx.x*1e-6f, c0=.1f,c1=.2f,c2=.3f,c3=.4f;
  for(int k=0;k<iters;k++){ c0=__expf(-c0)+a; c1=__expf(-c1)+a; c2=__expf(-c2)+a; c3=__expf(-c3)+a; }
  float s=c0+c1+c2+c3; if(s==1.2345f) out[0]=s;
}
int main(){
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t bytes = 8ull<<30; double2* p; CK(cudaMalloc(&p, bytes)); double* o; CK(cudaMalloc(&o, 64));
  size_t n2 = bytes/16; cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int grids[3] = {sms*4, sms*8, sms*16};
  for(int g: grids){
    wr<<<g,256>>>(p,n2,1.0); CK(cudaDeviceSynchronize());
    float best=1e9; for(int r=0;r<5;r++){cudaEventRecord(e0); wr<<<g,256>>>(p,n2,1.0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    printf("write-only   grid %5d: %.1f GB/s\n", g, bytes/best/1e6);
    best=1e9; for(int r=0;r<5;r++){cudaEventRecord(e0); wr_cs<<<g,256>>>(p,n2,1.0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    printf("write-only cs grid %5d: %.1f GB/s\n", g, bytes/best/1e6);
    best=1e9; for(int r=0;r<5;r++){cudaEventRecord(e0); rd<<<g,256>>>(p,n2,o); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    printf("read-only    grid %5d: %.1f GB/s\n", g, bytes/best/1e6);
  }
  int it=20000; dfma<<<sms*8,256>>>(o,10); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); dfma<<<sms*8,256>>>(o,it); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  double fl = 2.0*8*it*(double)sms*8*256; printf("fp64 fma: %.2f TFLOP/s\n", fl/ms/1e9);
  ex2f<<<sms*8,256>>>((float*)o,10); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); ex2f<<<sms*8,256>>>((float*)o,it); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("ex2.approx(+add): %.3f Tops/s\n", 4.0*it*(double)sms*8*256/ms/1e9);
  return 0;
}
