#include <cstdio>
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c){
  unsigned long long A=*(unsigned long long*)&a,B=*(unsigned long long*)&b,C=*(unsigned long long*)&c,D;
  asm("fma.rn.f32x2 %0,%1,%2,%3;":"=l"(D):"l"(A),"l"(B),"l"(C));
  return *(float2*)&D;
}
__global__ void k2(float* o, float p, int n){
  float2 a[8]; for(int i=0;i<8;i++) a[i]=make_float2(threadIdx.x*1e-3f+i, i*0.5f);
  float2 pp=make_float2(p,p*0.9f); float2 x=make_float2(0.1f,0.2f);
  for(int it=0;it<n;it++){
#pragma unroll
    for(int i=0;i<8;i++) a[i]=fma2(pp,a[i],x);
  }
  float s=0; for(int i=0;i<8;i++) s+=a[i].x+a[i].y; o[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k1(float* o, float p, int n){
  float a[16]; for(int i=0;i<16;i++) a[i]=threadIdx.x*1e-3f+i;
  float q=p*0.9f;
  for(int it=0;it<n;it++){
#pragma unroll
    for(int i=0;i<16;i++) a[i]=fmaf((i&1)?q:p,a[i],0.1f+ (i&1)*0.1f);
  }
  float s=0; for(int i=0;i<16;i++) s+=a[i]; o[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float*o; cudaMalloc(&o, 148*8*256*4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int n=20000;
  for(int rep=0;rep<2;rep++){
  for(int w=0;w<2;w++){
    cudaEventRecord(e0);
    if(w) k2<<<148*8,256>>>(o,0.99f,n); else k1<<<148*8,256>>>(o,0.99f,n);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fmas=148.0*8*256*16*(double)n;
    printf("%s: %.3f ms %.2f TFMA/s\n", w?"FFMA2":"FFMA", ms, fmas/ms/1e9);
  }}
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
