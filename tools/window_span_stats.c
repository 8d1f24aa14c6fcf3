// Analysis (not product): column-span / product statistics of the planner's greedy windows
// over cfg5's heavy rows.  Inputs: /tmp/rp.bin, /tmp/ci.bin (cfg5 CSR).
// build: gcc -O3 -fopenmp window_span_stats.c; run: ./a.out LOG_BIN_WIDTH CAP
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
#include <omp.h>
int64_t *rp; int32_t *ci; int64_t n;
int main(int argc, char** argv){
  int LOGW = argc>1? atoi(argv[1]):12; int CAPG = argc>2? atoi(argv[2]):3072;
  n = 4194304; rp = malloc((n+1)*8); ci = malloc(67092960ll*4);
  FILE*f=fopen("/tmp/rp.bin","rb"); fread(rp,8,n+1,f); fclose(f);
  f=fopen("/tmp/ci.bin","rb"); fread(ci,4,rp[n],f); fclose(f);
  int nb = (int)((n + (1<<LOGW)-1) >> LOGW);
  // span/products ratio buckets (products-weighted), and cf per window
  double wsum[16]={0}, wout[16]={0}; long wcnt[16]={0};
  double tot_heavy=0, tot_light=0, tot_out_heavy=0;
  #pragma omp parallel
  {
    int32_t* hist = calloc(nb,4); uint32_t* bm = calloc((n+31)/32,4);
    double l_ws[16]={0}, l_wo[16]={0}; long l_wc[16]={0}; double th=0, tl=0, toh=0;
    #pragma omp for schedule(dynamic,64)
    for (int64_t i=0;i<n;i++){
      int64_t P=0; for(int64_t p=rp[i];p<rp[i+1];p++){int k=ci[p]; P+=rp[k+1]-rp[k];}
      if (P<=4096){ tl+=P; continue; }
      th+=P;
      memset(hist,0,nb*4);
      for(int64_t p=rp[i];p<rp[i+1];p++){int k=ci[p]; for(int64_t q=rp[k];q<rp[k+1];q++){hist[ci[q]>>LOGW]++; bm[ci[q]>>5] |= 1u<<(ci[q]&31);} }
      // greedy windows
      int b=0;
      while(b<nb){
        int b0=b; int acc=hist[b]; b++;
        if (acc<=CAPG) while(b<nb && hist[b]<=CAPG && acc+hist[b]<=CAPG){acc+=hist[b]; b++;}
        if(acc==0) continue;
        int64_t c0=(int64_t)b0<<LOGW, c1=(int64_t)b<<LOGW; if(c1>n)c1=n;
        int64_t outs=0; for(int64_t w=c0/32; w<(c1+31)/32; w++) outs+=__builtin_popcount(bm[w]);
        double ratio=(double)(c1-c0)/acc; int bk=0; while(bk<15 && ratio > (1<<bk)*0.5) bk++;
        l_ws[bk]+=acc; l_wo[bk]+=outs; l_wc[bk]++; toh+=outs;
      }
      // clear bitmap
      for(int64_t p=rp[i];p<rp[i+1];p++){int k=ci[p]; for(int64_t q=rp[k];q<rp[k+1];q++) bm[ci[q]>>5]=0;}
    }
    #pragma omp critical
    { for(int j=0;j<16;j++){wsum[j]+=l_ws[j]; wout[j]+=l_wo[j]; wcnt[j]+=l_wc[j];} tot_heavy+=th; tot_light+=tl; tot_out_heavy+=toh; }
  }
  printf("LOGW=%d CAPG=%d heavy products %.3e light %.3e heavy outputs %.3e\n",LOGW,CAPG,tot_heavy,tot_light,tot_out_heavy);
  for(int j=0;j<16;j++) if(wcnt[j]) printf("span/prod <= %8.1f : windows %9ld products %.3e (%.1f%%) outputs %.3e cf %.3f\n",(1<<j)*0.5,wcnt[j],wsum[j],100*wsum[j]/tot_heavy,wout[j],wsum[j]/wout[j]);
}
