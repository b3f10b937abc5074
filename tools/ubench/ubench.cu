// Microbenchmarks for B200 design decisions: FP64 pipe, conversions, HBM write/copy.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
constexpr int ITERS = 4096;
__global__ void k_dfma(double* out, double a, double b) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<ITERS;i++){ x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b); x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);}
  if (x0+x1+x2+x3+x4+x5+x6+x7 == 12345.0) out[0]=1;
}
__global__ void k_dadd(double* out, double a) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<ITERS;i++){ x0+=a; x1+=a; x2+=a; x3+=a; x4+=a; x5+=a; x6+=a; x7+=a; }
  if (x0+x1+x2+x3+x4+x5+x6+x7 == 12345.0) out[0]=1;
}
__global__ void k_ffma(float* out, float a, float b) {
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<ITERS;i++){ x0=fmaf(x0,a,b); x1=fmaf(x1,a,b); x2=fmaf(x2,a,b); x3=fmaf(x3,a,b); x4=fmaf(x4,a,b); x5=fmaf(x5,a,b); x6=fmaf(x6,a,b); x7=fmaf(x7,a,b);}
  if (x0+x1+x2+x3+x4+x5+x6+x7 == 12345.0f) out[0]=1;
}
// float -> double conversion throughput (8 independent cvts per iter, cheap dependence through float add)
__global__ void k_f2d(double* out, float a) {
  float f0=threadIdx.x, f1=f0+1, f2=f0+2, f3=f0+3, f4=f0+4, f5=f0+5, f6=f0+6, f7=f0+7;
  double s0=0,s1=0;
  for (int i=0;i<ITERS;i++){
    double d0=(double)f0, d1=(double)f1, d2=(double)f2, d3=(double)f3, d4=(double)f4, d5=(double)f5, d6=(double)f6, d7=(double)f7;
    s0 = (d0>d1? d2: d3) + s0; s1 = (d4>d5? d6: d7) + s1;
    f0+=a; f1+=a; f2+=a; f3+=a; f4+=a; f5+=a; f6+=a; f7+=a;
  }
  if (s0+s1 == 12345.0) out[0]=1;
}
__global__ void k_d2f(float* out, double a) {
  double d0=threadIdx.x, d1=d0+1, d2=d0+2, d3=d0+3, d4=d0+4, d5=d0+5, d6=d0+6, d7=d0+7;
  float s0=0,s1=0;
  for (int i=0;i<ITERS;i++){
    float f0=(float)d0, f1=(float)d1, f2=(float)d2, f3=(float)d3, f4=(float)d4, f5=(float)d5, f6=(float)d6, f7=(float)d7;
    s0 += fmaxf(fmaxf(f0,f1),fmaxf(f2,f3)); s1 += fmaxf(fmaxf(f4,f5),fmaxf(f6,f7));
    d0+=a; d1+=a; d2+=a; d3+=a; d4+=a; d5+=a; d6+=a; d7+=a;
  }
  if (s0+s1 == 12345.0f) out[0]=1;
}
__global__ void k_ddiv(double* out, double a) {
  double x0=threadIdx.x+1, x1=x0+1, x2=x0+2, x3=x0+3;
  for (int i=0;i<ITERS/16;i++){ x0=a/x0; x1=a/x1; x2=a/x2; x3=a/x3; }
  if (x0+x1+x2+x3 == 12345.0) out[0]=1;
}
__global__ void k_write(float4* p, size_t n) {
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st = (size_t)gridDim.x*blockDim.x;
  for (; i<n; i+=st) p[i] = make_float4(1,2,3,4);
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st = (size_t)gridDim.x*blockDim.x;
  for (; i<n; i+=st) b[i] = a[i];
}
// read 4B, write 24B per element (the fused-pass traffic shape), coalesced float2 stores
__global__ void k_r4w24(const float* __restrict__ a, float2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; size_t st = (size_t)gridDim.x*blockDim.x;
  for (; i<n; i+=st) { float v=a[i]; b[3*i]=make_float2(v,v); b[3*i+1]=make_float2(v,v); b[3*i+2]=make_float2(v,v);} 
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  double* dout; float* fout; CK(cudaMalloc(&dout, 64)); CK(cudaMalloc(&fout, 64));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms*8, thr=256; double nthr = (double)blocks*thr;
  auto timeit=[&](auto f, const char* name, double ops_per_thread){
    f(); cudaDeviceSynchronize(); float best=1e9;
    for(int r=0;r<5;r++){ cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    double ops = nthr*ops_per_thread; double per_s = ops/(best*1e-3);
    printf("%-8s %8.3f ms  %10.2f Gops/s  %6.1f ops/clk/SM(at %d MHz)\n", name, best, per_s/1e9, per_s/(sms*(clk*1e3)), clk/1000);
  };
  timeit([&]{k_dfma<<<blocks,thr>>>(dout,1.0000001,1e-9);}, "DFMA", 8.0*ITERS);
  timeit([&]{k_dadd<<<blocks,thr>>>(dout,1e-9);}, "DADD", 8.0*ITERS);
  timeit([&]{k_ffma<<<blocks,thr>>>(fout,1.0000001f,1e-9f);}, "FFMA", 8.0*ITERS);
  timeit([&]{k_f2d<<<blocks,thr>>>(dout,1e-3f);}, "F2D", 8.0*ITERS);
  timeit([&]{k_d2f<<<blocks,thr>>>(fout,1e-3);}, "D2F", 8.0*ITERS);
  timeit([&]{k_ddiv<<<blocks,thr>>>(dout,3.0);}, "DDIV", 4.0*ITERS/16);
  size_t bytes = (size_t)4<<30; size_t n = bytes/16; float4 *a,*b; CK(cudaMalloc(&a,bytes)); CK(cudaMalloc(&b,bytes));
  cudaMemset(a,0,bytes); cudaMemset(b,0,bytes);
  auto bw=[&](auto f, const char* name, double by){
    f(); cudaDeviceSynchronize(); float best=1e9;
    for(int r=0;r<5;r++){ cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    printf("%-8s %8.3f ms  %8.1f GB/s\n", name, best, by/(best*1e-3)/1e9);
  };
  bw([&]{k_write<<<sms*16,256>>>(b,n);}, "write", (double)bytes);
  bw([&]{k_copy<<<sms*16,256>>>(a,b,n/2);}, "copy", (double)bytes);  // n/2 float4 read + write = bytes total
  size_t npx = bytes/28; 
  bw([&]{k_r4w24<<<sms*16,256>>>((const float*)a,(float2*)b,npx);}, "r4w24", (double)npx*28);
  bw([&]{cudaMemcpyAsync(b,a,bytes/2,cudaMemcpyDeviceToDevice);}, "memcpy", (double)bytes);
  printf("done\n");
  return 0;
}
