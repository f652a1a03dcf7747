#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
static const uint64_t T[32] = {
#include "tab.inc"
};
static inline uint64_t asu64(double d){uint64_t u;memcpy(&u,&d,8);return u;}
static inline double asd(uint64_t u){double d;memcpy(&d,&u,8);return d;}
static inline uint32_t asu32(float f){uint32_t u;memcpy(&u,&f,4);return u;}
#define N 32
static const double InvLn2N = 0x1.71547652b82fep+0 * N;
static const double SHIFT = 0x1.8p+52;
static const double C0 = 0x1.c6af84b912394p-5/N/N/N, C1 = 0x1.ebfce50fac4f3p-3/N/N, C2 = 0x1.62e42ff0c52d6p-1/N;
// variant bits: 1 = fma for poly, 2 = fma for kd, 4 = fma for r
static float myexpf(float x, int var){
  double xd = x;
  uint32_t abstop = (asu32(x) >> 20) & 0x7ff;
  if (abstop >= (asu32(88.0f)>>20)) {
    if (asu32(x) == asu32(-INFINITY)) return 0.0f;
    if (abstop >= (asu32(INFINITY)>>20)) return x + x;
    if (x > 0x1.62e42ep6f) return INFINITY;
    if (x < -0x1.9fe368p6f) return 0.0f;
  }
  double z = InvLn2N * xd;
  double kd = (var&2) ? fma(InvLn2N, xd, SHIFT) : (z + SHIFT);
  uint64_t ki = asu64(kd);
  kd -= SHIFT;
  double r = (var&4) ? fma(InvLn2N, xd, -kd) : (z - kd);
  uint64_t t = T[ki % N];
  t += ki << (52 - 5);
  double s = asd(t);
  double y;
  if (var&1) {
    double zz = fma(C0, r, C1);
    double r2 = r*r;
    y = fma(C2, r, 1.0);
    y = fma(zz, r2, y);
  } else {
    double zz = C0*r + C1;
    double r2 = r*r;
    y = C2*r + 1.0;
    y = zz*r2 + y;
  }
  y = y * s;
  return (float)y;
}
int main(){
  long long bad[8]={0}; long long cnt=0;
  for (uint64_t u = 0; u < (1ull<<32); u += 1) {
    float x; uint32_t uu=(uint32_t)u; memcpy(&x,&uu,4);
    if (isnan(x)) continue;
    if (!(x > -110.0f && x < 90.0f)) continue;
    cnt++;
    float ref = expf(x);
    for (int v=0; v<8; v++) { float m = myexpf(x,v); if (asu32(m)!=asu32(ref)) bad[v]++; }
  }
  printf("count %lld\n",cnt);
  for(int v=0;v<8;v++) printf("var %d bad %lld\n", v, bad[v]);
}
