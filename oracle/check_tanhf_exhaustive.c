#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
static inline uint32_t fw(float f){uint32_t u;memcpy(&u,&f,4);return u;}
static inline float wf(uint32_t u){float f;memcpy(&f,&u,4);return f;}
static const float one=1.0f, huge=1.0e+30f, tiny=1.0e-30f,
 o_threshold=8.8721679688e+01f, ln2_hi=6.9313812256e-01f, ln2_lo=9.0580006145e-06f, invln2=1.4426950216e+00f;
static float Q1=-3.3333335072e-02f,Q2=1.5873016091e-03f,Q3=-7.9365076090e-05f,Q4=4.0082177293e-06f,Q5=-2.0109921195e-07f;
static int two_coef = 0;
static float myexpm1f(float x){
  float y,hi,lo,c=0,t,e,hxs,hfx,r1; int32_t k,xsb; uint32_t hx=fw(x);
  xsb = hx&0x80000000; hx &= 0x7fffffff;
  if(hx >= 0x4195b844) {
    if(hx >= 0x42b17218) { if(hx>0x7f800000) return x+x; if(hx==0x7f800000) return (xsb==0)?x:-1.0f; if(x>o_threshold) return huge*huge; }
    if(xsb!=0) return tiny-one;
  }
  if(hx > 0x3eb17218) {
    if(hx < 0x3F851592) { if(xsb==0){hi=x-ln2_hi;lo=ln2_lo;k=1;} else {hi=x+ln2_hi;lo=-ln2_lo;k=-1;} }
    else { k = invln2*x+((xsb==0)?0.5f:-0.5f); t=k; hi=x-t*ln2_hi; lo=t*ln2_lo; }
    x = hi-lo; c=(hi-x)-lo;
  } else if(hx < 0x33000000) { t=huge+x; return x-(t-(huge+x)); }
  else k=0;
  hfx=0.5f*x; hxs=x*hfx;
  if (two_coef) r1 = one+hxs*(Q1+hxs*Q2);
  else r1=one+hxs*(Q1+hxs*(Q2+hxs*(Q3+hxs*(Q4+hxs*Q5))));
  t=3.0f-r1*hfx; e=hxs*((r1-t)/(6.0f-x*t));
  if(k==0) return x-(x*e-hxs);
  e=(x*(e-c)-c); e-=hxs;
  if(k==-1) return 0.5f*(x-e)-0.5f;
  if(k==1){ if(x<-0.25f) return -2.0f*(e-(x+0.5f)); else return one+2.0f*(x-e); }
  if(k<=-2||k>56){ y=one-(e-x); uint32_t i=fw(y); y=wf(i+(k<<23)); return y-one; }
  t=one;
  if(k<23){ t=wf(0x3f800000-(0x1000000>>k)); y=t-(e-x); uint32_t i=fw(y); y=wf(i+(k<<23)); }
  else { t=wf((0x7f-k)<<23); y=x-(e+t); y+=one; uint32_t i=fw(y); y=wf(i+(k<<23)); }
  return y;
}
static float mytanhf(float x){
  float t,z; int32_t jx=(int32_t)fw(x), ix=jx&0x7fffffff;
  if(ix>=0x7f800000){ if(jx>=0) return one/x+one; else return one/x-one; }
  if(ix<0x41b00000){
    if(ix==0) return x;
    if(ix<0x24000000) return x*(one+x);
    if(ix>=0x3f800000){ t=myexpm1f(2.0f*fabsf(x)); z=one-2.0f/(t+2.0f); }
    else { t=myexpm1f(-2.0f*fabsf(x)); z=-t/(t+2.0f); }
  } else z=one-tiny;
  return (jx>=0)?z:-z;
}
int main(int argc,char**argv){
  if (argc>1) { two_coef=1; Q1=-3.3333212137e-2f; Q2=1.5807170421e-3f; }
  long long bad=0, badm=0;
  for (uint64_t u=0; u<0x7f800000ull; u+=1){
    float x=wf((uint32_t)u);
    if (fw(mytanhf(x))!=fw(tanhf(x))) bad++;
    if (fw(mytanhf(-x))!=fw(tanhf(-x))) bad++;
    if ((u & 15)==0 && fw(myexpm1f(x))!=fw(expm1f(x))) badm++;
    if ((u & 15)==0 && fw(myexpm1f(-x))!=fw(expm1f(-x))) badm++;
  }
  printf("two_coef=%d tanh bad %lld expm1(sampled) bad %lld\n", two_coef, bad, badm);
}
