// Analysis (not product): CPU model of the counting sort's rank-loop cost over the
// greedy windows of cfg5's heavy rows (warp-iterations per product for 2^NBL buckets).
// Inputs: /tmp/rp.bin (int64 row_ptr) and /tmp/ci.bin (int32 col_idx) of cfg5.
// build: gcc -O3 window_bucket_model.c; run: ./a.out NBL stride
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
int64_t *rp; int32_t *ci; int64_t n;
static int bl(uint32_t x){ return x? 32-__builtin_clz(x):0; }
int main(int argc,char**argv){
  int NBL = argc>1? atoi(argv[1]):11; int stride = argc>2? atoi(argv[2]):64;
  n=4194304; rp=malloc((n+1)*8); ci=malloc(67092960ll*4);
  FILE*f=fopen("/tmp/rp.bin","rb"); if(fread(rp,8,n+1,f)){}; fclose(f);
  f=fopen("/tmp/ci.bin","rb"); if(fread(ci,4,rp[n],f)){}; fclose(f);
  int nb=1024; int32_t*hist=calloc(nb,4); uint32_t*keys=malloc(1<<24); int NB=1<<NBL;
  int *cnt=calloc(NB+1,4), *start=calloc(NB+1,4); int *bucket_of=malloc(4096*4*8);
  double prod=0, iters=0, iters_el=0, dups=0; long wins=0; double maxb_sum=0;
  int hrow=0;
  for(int64_t i=0;i<n;i++){
    int64_t P=0; for(int64_t p=rp[i];p<rp[i+1];p++){int k=ci[p]; P+=rp[k+1]-rp[k];}
    if(P<=4096) continue; if((hrow++)%stride) continue;
    memset(hist,0,nb*4);
    for(int64_t p=rp[i];p<rp[i+1];p++){int k=ci[p]; for(int64_t q=rp[k];q<rp[k+1];q++) hist[ci[q]>>12]++;}
    int b=0;
    while(b<nb){
      int b0=b, acc=hist[b]; b++;
      if(acc<=3072) while(b<nb && hist[b]<=3072 && acc+hist[b]<=3072){acc+=hist[b]; b++;}
      if(acc==0||acc>3072) continue;
      int c0=b0<<12, c1=b<<12; if(c1>n)c1=n;
      int t=0;
      for(int64_t p=rp[i];p<rp[i+1];p++){int k=ci[p]; for(int64_t q=rp[k];q<rp[k+1];q++){int c=ci[q]; if(c>=c0&&c<c1) keys[t++]=c-c0;}}
      int bits=bl((uint32_t)(c1-c0-1)); int sh=bits>NBL?bits-NBL:0;
      memset(cnt,0,(NB+1)*4);
      for(int e=0;e<t;e++) cnt[keys[e]>>sh]++;
      int s=0; for(int x=0;x<NB;x++){start[x]=s; s+=cnt[x];} start[NB]=s;
      // slot -> bucket
      for(int x=0;x<NB;x++) for(int q=start[x];q<start[x+1];q++) bucket_of[q]=x;
      int mb=0;
      for(int w=0; w<t; w+=32){ int m=1; for(int q=w;q<w+32&&q<t;q++){int sz=cnt[bucket_of[q]]; if(sz>1&&sz>m)m=sz;} iters+=m; }
      for(int x=0;x<NB;x++){ if(cnt[x]>1) iters_el+= (double)cnt[x]*cnt[x]; if(cnt[x]>mb)mb=cnt[x]; }
      maxb_sum+=mb;
      prod+=t; wins++;
    }
  }
  printf("NB=2^%d windows %ld products %.3e  warp-iters/product %.3f  elem-iters/product %.2f  mean max bucket %.1f\n",NBL,wins,prod,iters/prod,iters_el/prod,maxb_sum/wins);
}
