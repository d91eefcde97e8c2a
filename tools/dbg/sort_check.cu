// debug: radix y-ordering (pip_sort.cu) on random points; checks permutation + order
#include "../../paper_2306_04316_b200/csrc/pip_kernels.h"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cstring>
static unsigned long long hkey(double v){ unsigned long long b; v = v + 0.0; memcpy(&b,&v,8); return (b>>63)? ~b : (b|0x8000000000000000ull);}
int main(int argc, char** argv){
  uint64_t n = argc>1? strtoull(argv[1],0,10) : 1000000;
  std::mt19937_64 rng(1); std::uniform_real_distribution<double> U(-1,1);
  std::vector<double> xy(2*n); for (auto& v: xy) v = U(rng);
  unsigned long long bb[8] = {hkey(-0.9), hkey(-1.0), ~hkey(0.9), ~hkey(1.0), 0,0,0,0};
  double *dp; unsigned long long* db; void* scr; uint32_t *sidx, *nin; double* spts;
  cudaMalloc(&dp, 16*n); cudaMemcpy(dp, xy.data(), 16*n, cudaMemcpyHostToDevice);
  cudaMalloc(&db, 64); cudaMemcpy(db, bb, 64, cudaMemcpyHostToDevice);
  cudaMalloc(&scr, pcd::bucket_scratch_bytes(n)); cudaMalloc(&sidx, 4*n); cudaMalloc(&nin, 4); cudaMalloc(&spts, 16*n);
  uint64_t L=0;
  pcd::BucketArgs a{dp, n, db, 1, scr, spts, sidx, nin};
  cudaError_t e = pcd::launch_bucket(a, 0, 0, &L); cudaDeviceSynchronize();
  printf("launch %s sync %s\n", cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  std::vector<uint32_t> h(n); uint32_t hn; cudaMemcpy(h.data(), sidx, 4*n, cudaMemcpyDeviceToHost); cudaMemcpy(&hn, nin, 4, cudaMemcpyDeviceToHost);
  uint64_t expect_in=0; for (uint64_t i=0;i<n;++i) if (xy[2*i]>=-0.9 && xy[2*i]<=0.9) ++expect_in;
  { uint64_t nt=(n+4095)/4096; size_t o=((n*2+15)/16*16)*2+((n*4+15)/16*16)+n*16;
    std::vector<uint32_t> cnt(2*256*nt), tot(512), base(512);
    cudaMemcpy(cnt.data(), (char*)scr+o, 4*cnt.size(), cudaMemcpyDeviceToHost); o += (2*256*nt*4+15)/16*16;
    cudaMemcpy(tot.data(), (char*)scr+o, 2048, cudaMemcpyDeviceToHost); o+=2048;
    cudaMemcpy(base.data(), (char*)scr+o, 2048, cudaMemcpyDeviceToHost);
    uint64_t st0=0, st1=0; for(int d=0;d<256;++d){st0+=tot[d]; st1+=tot[256+d];}
    printf("nt %llu sum tot pass0 %llu pass1 %llu base1[255] %u base0[255] %u tot1[255] %u\n",(unsigned long long)nt,(unsigned long long)st0,(unsigned long long)st1,base[511],base[255],tot[511]);
    for (int d=250; d<256; ++d) printf("d%d: tot1 %u base1 %u | ", d, tot[256+d], base[256+d]); printf("\n");
  }
  printf("n_in %u expect %llu\n", hn, (unsigned long long)expect_in);
  { std::vector<double> hp(2*n); cudaMemcpy(hp.data(), spts, 16*n, cudaMemcpyDeviceToHost); uint64_t bad=0;
    for (uint64_t i=0;i<n;++i) if (h[i]<n && (hp[2*i]!=xy[2*h[i]] || hp[2*i+1]!=xy[2*h[i]+1])) ++bad; printf("point mismatches %llu\n",(unsigned long long)bad); }
  std::vector<char> seen(n,0); uint64_t dup=0, oob=0;
  for (uint64_t i=0;i<n;++i){ if (h[i]>=n){++oob;continue;} if (seen[h[i]]) ++dup; seen[h[i]]=1; }
  uint64_t inv=0; double prev=-1e300;
  for (uint64_t i=0;i<hn && i<n;++i){ uint32_t j=h[i]; if (j>=n) continue; double y = xy[2*j+1]; double ky=floor((y+1.0)*65280/2.0); if (ky<prev) ++inv; prev=ky; }
  printf("dup %llu oob %llu inversions %llu\n",(unsigned long long)dup,(unsigned long long)oob,(unsigned long long)inv);
  for (int i=0;i<10;++i) printf("%u(%.4f) ", h[i], xy[2*h[i]+1]); printf("\n");
  return 0;
}
