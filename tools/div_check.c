/* Checks that the reciprocal product plus one FMA remainder correction used by
   line_kernels.cu (div_rcp) returns the correctly rounded quotient x / d for the
   Lagrange denominators and grid spacings 1/(n-1): gcc -O2 -ffp-contract=off
   tools/div_check.c -lm && ./a.out   (prints "bad 0 of 1000000000") */
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
static uint64_t s=88172645463325252ull;
static inline uint64_t xr(){s^=s<<13;s^=s>>7;s^=s<<17;return s;}
static inline double rnd(double lo,double hi){return lo+(hi-lo)*(xr()>>11)*(1.0/9007199254740992.0);}
int main(){
  double dens[]={24,-6,4,6,-24,2,-2,120,-30,20,12,-12,36,-144,720,-120,48,-48,240,-240, 255.0, 127.0, 63.0, 191.0, 47.0};
  long bad=0,tot=0;
  for(int di=0;di<25;di++){
    double d = dens[di]; if(di>=20) d = 1.0/dens[di];   /* grid spacing h = 1/(n-1) */
    double r = 1.0/d;
    for(long i=0;i<40000000;i++){
      double x = (di>=20)? rnd(0.0,1.0) : rnd(-3.0,3.0)*pow(2.0,(double)((int)(xr()%40)-20));
      double q0 = x*r;
      double rem = fma(-q0,d,x);
      double q1 = fma(rem,r,q0);
      double ex = x/d;
      tot++; if(q1!=ex){bad++; if(bad<5) printf("d=%g x=%.17g q1=%.17g ex=%.17g\n",d,x,q1,ex);}
    }
  }
  printf("bad %ld of %ld\n",bad,tot);
}
