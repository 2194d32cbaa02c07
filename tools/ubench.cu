// Throughput microbenchmarks for design decisions (not part of the product).
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096
__global__ void k_dfma(double* o, double s){ double a[8]; for(int k=0;k<8;k++) a[k]=s+threadIdx.x+k;
  for(int i=0;i<N_IT;i++){
#pragma unroll

    for(int k=0;k<8;k++) a[k]=__fma_rn(a[k],0.999999,1e-9);} double r=0; for(int k=0;k<8;k++) r+=a[k]; if(r==1.2345) o[0]=r; }
__global__ void k_f2i(double* o, double s){ double a[8]; int acc=0; for(int k=0;k<8;k++) a[k]=s*(threadIdx.x+k);
  for(int i=0;i<N_IT;i++){
#pragma unroll

    for(int k=0;k<8;k++){ acc += __double2int_rz(a[k]); a[k] = __longlong_as_double(__double_as_longlong(a[k]) ^ (acc & 1)); } }
  if(acc==12345) o[0]=acc; }
__global__ void k_dsetp(double* o, double s){ double a[8]; int acc=0; for(int k=0;k<8;k++) a[k]=s*(threadIdx.x+k);
  for(int i=0;i<N_IT;i++){
#pragma unroll

    for(int k=0;k<8;k++){ acc += (a[k] < s) ; a[k] = __longlong_as_double(__double_as_longlong(a[k]) + 1); } }
  if(acc==12345) o[0]=acc; }
__global__ void k_f2f(double* o, double s){ double a[8]; float acc=0; for(int k=0;k<8;k++) a[k]=s*(threadIdx.x+k);
  for(int i=0;i<N_IT;i++){
#pragma unroll

    for(int k=0;k<8;k++){ acc += __double2float_rn(a[k]); a[k] = __longlong_as_double(__double_as_longlong(a[k]) + 1); } }
  if(acc==12345) o[0]=acc; }
__global__ void k_iadd(double* o, double s){ unsigned a[8]; for(int k=0;k<8;k++) a[k]=threadIdx.x+k;
  for(int i=0;i<N_IT;i++){
#pragma unroll

    for(int k=0;k<8;k++){ a[k] = (a[k] ^ (a[k]>>3)) + 0x9e3779b9u; } }
  unsigned r=0; for(int k=0;k<8;k++) r+=a[k]; if(r==12345) o[0]=r; }
__global__ void k_smem64(double* o, double s){ __shared__ long long h[16*256]; for(int b=0;b<16;b++) h[b*256+threadIdx.x]=0;
  unsigned st=threadIdx.x*2654435761u;
  for(int i=0;i<N_IT;i++){
#pragma unroll

    for(int k=0;k<8;k++){ st = st*1664525u+1013904223u; int b=(st>>28); h[b*256+threadIdx.x] += (long long)st; } }
  long long r=0; for(int b=0;b<16;b++) r+=h[b*256+threadIdx.x]; if(r==12345) o[0]=r; }
int main(){ double* o; cudaMalloc(&o, 8); cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks=148*8, thr=256; double ops=(double)blocks*thr*N_IT*8;
  const char* names[]={"dfma","f2i.f64","dsetp","f2f.f32.f64","iadd/lop (2 ops)","smem int64 RMW (1 upd)"};
  void (*ks[])(double*,double)={k_dfma,k_f2i,k_dsetp,k_f2f,k_iadd,k_smem64};
  for(int t=0;t<6;t++){ for(int rep=0;rep<2;rep++){ cudaEventRecord(a); ks[t]<<<blocks,thr>>>(o,1.5); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); if(rep) printf("%-24s %8.3f ms  %8.1f Gop/s  %6.1f ops/clk/SM@1.965GHz\n", names[t], ms, ops/ms/1e6, ops/(ms*1e-3)/148/1.965e9); } }
  return 0; }
