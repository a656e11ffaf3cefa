/* Sequential model of the key set's bucketized insert (kernels.cuh scan_cset_kernel,
 * cset_resolve_bucket): random 48-bit keys (cip << 16 | bucket), the same perm48, 4-entry
 * buckets, linear overflow into the next bucket up to a bucket limit.  Prints the largest
 * displacement, the keys that overflowed the limit and the displacement histogram.
 *   gcc -O2 -o tools/bin/keyset_sim tools/keyset_sim.c
 *   tools/bin/keyset_sim <log2 entries> <keys> <bucket bits> <bucket limit>
 * profiles/r02_ab_keyset.md uses it to size kCsetBucketLimit. */
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
static uint64_t perm48(uint64_t x){const uint64_t M=(1ull<<48)-1;
 x=(x*0x9E3779B97F4Bull)&M; x^=x>>23; x=(x*0xC2B2AE3D27D5ull)&M; x^=x>>25; x=(x*0x165667B19E37ull)&M; x^=x>>24; return x;}
static uint64_t s=88172645463325252ull; static uint64_t rnd(){s^=s<<13;s^=s>>7;s^=s<<17;return s;}
int main(int argc,char**argv){int lg=atoi(argv[1]); long n=atol(argv[2]); int bbits=atoi(argv[3]);
 int LB=2,BW=4; uint32_t lgb=lg-LB, rb=48-lgb, bmask=(1u<<lgb)-1; uint32_t*t=calloc((size_t)1<<lg,4);
 long over=0; int dmax=0; long hist[64]={0};
 for(long i=0;i<n;i++){uint64_t key=((rnd()&0xffffffffull)<<16)|(rnd()&((1ull<<bbits)-1)); uint64_t x=perm48(key);
  uint32_t hb=x>>rb, rem=x&((1u<<rb)-1); int done=0;
  for(uint32_t d=0; d<(uint32_t)atoi(argv[4]) && !done; d++){uint32_t want=(d+1)<<rb|rem; uint32_t*b=t+(size_t)((hb+d)&bmask)*BW;
   for(int j=0;j<BW;j++){ if(b[j]==want){done=2;break;} if(b[j]==0){b[j]=want;done=1;hist[d]++; if((int)d>dmax)dmax=d;break;} } }
  if(!done) over++; }
 printf("lg %d n %ld load %.3f dmax %d overflow %ld  hist:",lg,n,(double)n/(1l<<lg),dmax,over); for(int d=0;d<8;d++)printf(" %ld",hist[d]); printf("\n"); }
