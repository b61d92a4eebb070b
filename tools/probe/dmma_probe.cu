#include <cstdio>
__global__ void k884(double* o, int it){
  double a=threadIdx.x*1e-3, b=1.0001, c0=0,c1=0, d0=0,d1=0,e0=0,e1=0,f0=0,f1=0;
  for(int i=0;i<it;i++){
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0),"+d"(c1) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0),"+d"(d1) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(e0),"+d"(e1) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(f0),"+d"(f1) : "d"(a),"d"(b));
  }
  if(c0+c1+d0+d1+e0+e1+f0+f1==1.234) o[0]=c0;
}
__global__ void k1684(double* o, int it){
  double a0=threadIdx.x*1e-3,a1=a0+1, b=1.0001, c[4][4]={};
  for(int i=0;i<it;i++){
    #pragma unroll
    for(int j=0;j<4;j++)
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};" : "+d"(c[j][0]),"+d"(c[j][1]),"+d"(c[j][2]),"+d"(c[j][3]) : "d"(a0),"d"(a1),"d"(b));
  }
  double s=0; for(int j=0;j<4;j++) for(int q=0;q<4;q++) s+=c[j][q]; if(s==1.234) o[0]=s;
}
__global__ void k16816(double* o, int it){
  double a[8], bb[4], c[4][4]={};
  for(int q=0;q<8;q++) a[q]=threadIdx.x*1e-3+q; for(int q=0;q<4;q++) bb[q]=1.0001+q*1e-9;
  for(int i=0;i<it;i++){
    #pragma unroll
    for(int j=0;j<4;j++)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};" : "+d"(c[j][0]),"+d"(c[j][1]),"+d"(c[j][2]),"+d"(c[j][3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),"d"(bb[0]),"d"(bb[1]),"d"(bb[2]),"d"(bb[3]));
  }
  double s=0; for(int j=0;j<4;j++) for(int q=0;q<4;q++) s+=c[j][q]; if(s==1.234) o[0]=s;
}
__global__ void kdfma(double* o, int it){
  double a=threadIdx.x*1e-3, b=1.0000001, c[8]={.1,.2,.3,.4,.5,.6,.7,.8};
  for(int k=0;k<it;k++){ for(int j=0;j<8;j++) c[j]=fma(c[j],b,a);} double s=0; for(int j=0;j<8;j++) s+=c[j]; if(s==1.2345) o[0]=s;
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, 64); cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int it=20000; int g=sms*4, b=256;
  #define RUN(K, FMAS_PER_ITER_PER_WARP, NAME) K<<<g,b>>>(o,10); cudaDeviceSynchronize(); cudaEventRecord(e0); K<<<g,b>>>(o,it); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); \
    printf("%-10s %.2f TFLOP/s (%s)\n", NAME, 2.0*FMAS_PER_ITER_PER_WARP*it*(double)g*(b/32)/ms/1e9, cudaGetErrorString(cudaGetLastError()));
  RUN(kdfma, 8*32, "dfma");
  RUN(k884, 4*256, "m8n8k4");
  RUN(k1684, 4*512, "m16n8k4");
  RUN(k16816, 4*2048, "m16n8k16");
  return 0;
}
