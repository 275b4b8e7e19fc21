/* tools/libm_exhaustive.c: full 2^32 sweep of oracle/libm_port.c (both ifunc variants)
   against the live glibc log10f / powf(10, y).  Build: gcc -O2 tools/libm_exhaustive.c
   oracle/_ref/libm_port.o -lm.  Result recorded in DESIGN.md. */
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
float oracle_log10f(float, int); float oracle_powf(float, float, int);
int main(){
  uint64_t bad_l[2]={0,0}, bad_p[2]={0,0}, n=0;
  for (uint64_t u=0; u<(1ull<<32); u+=1) { uint32_t b=(uint32_t)u; float x; memcpy(&x,&b,4);
    n++;
    if (!(x>0) || isinf(x)) { } else {
      float g=log10f(x);
      for(int v=0; v<2; ++v){ float o=oracle_log10f(x,v); if (memcmp(&g,&o,4)) bad_l[v]++; }
    }
    float gp=powf(10.0f,x);
    for(int v=0; v<2; ++v){ float op=oracle_powf(10.0f,x,v); if (memcmp(&gp,&op,4) && !(isnan(gp)&&isnan(op))) bad_p[v]++; }
  }
  printf("n=%lu log10f mismatches: sse2=%lu fma=%lu; powf mismatches: sse2=%lu fma=%lu\n", n, bad_l[0], bad_l[1], bad_p[0], bad_p[1]);
}
