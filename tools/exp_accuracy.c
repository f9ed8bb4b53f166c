#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include "tab.h"
static double fexp(double x) {
    if (x < -708.3) return x < -745.2 ? 0.0 : exp(x);
    const double magic = 6755399441055744.0; /* 1.5*2^52 */
    double kd = fma(x, INV_LN2_64, magic);
    int64_t kb; memcpy(&kb, &kd, 8);
    int k = (int)(int32_t)(uint32_t)kb;
    kd -= magic;
    double r = fma(kd, -LN2_64_HI, x);
    r = fma(kd, -LN2_64_LO, r);
    double q = fma(r, 1.0/120.0, 1.0/24.0);
    q = fma(q, r, 1.0/6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    double rq = r * q;
    double t = TAB[k & 63];
    double y = fma(t, rq, t);
    int m = k >> 6;
    uint64_t yb; memcpy(&yb, &y, 8);
    yb += (uint64_t)(int64_t)m << 52;
    memcpy(&y, &yb, 8);
    return y;
}
int main(){
    double maxulp=0, worstx=0; long bad=0;
    srand(1);
    for (long i=0;i<20000000;i++){
        double x = -745.0 * ((double)rand()/RAND_MAX);
        if (i%3==0) x = -5.0*((double)rand()/RAND_MAX);
        if (i%7==0) x = -1e-3*((double)rand()/RAND_MAX);
        double a = fexp(x), b = exp(x);
        if (b == 0) continue;
        double ulp = fabs(a-b)/ (nextafter(b, INFINITY)-b);
        if (ulp > maxulp){maxulp=ulp; worstx=x;}
        if (ulp > 1.0) bad++;
    }
    printf("max ulp vs glibc %.3f at x=%.17g ; >1ulp count %ld\n", maxulp, worstx, bad);
    printf("exp(0)=%.17g exp(-1)=%.17g\n", fexp(0.0), fexp(-1.0));
}
