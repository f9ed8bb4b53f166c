#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include "exp_tab256.h"
static double fexp(double x) {
    const double magic = 6755399441055744.0;
    double kd = fma(x, L2E256, magic);
    int64_t kb; memcpy(&kb, &kd, 8);
    int k = (int)(int32_t)(uint32_t)kb;
    kd -= magic;
    double r = fma(kd, -LN2_256, x);
    double q = fma(r, 1.0/24.0, 1.0/6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    double t = TAB[k & 255];
    double y = fma(t, r * q, t);
    int m = k >> 8;
    uint64_t yb; memcpy(&yb, &y, 8);
    yb += (uint64_t)(int64_t)m << 52;
    memcpy(&y, &yb, 8);
    return y;
}
int main(){
    double maxrel=0, worstx=0, maxulp_small=0;
    srand(1);
    for (long i=0;i<20000000;i++){
        double x = -708.0 * ((double)rand()/RAND_MAX);
        if (i%3==0) x = -5.0*((double)rand()/RAND_MAX);
        if (i%7==0) x = -1e-3*((double)rand()/RAND_MAX);
        double a = fexp(x), b = exp(x);
        double rel = fabs(a-b)/b;
        if (rel > maxrel){maxrel=rel; worstx=x;}
        if (x > -5) { double u = fabs(a-b)/(nextafter(b,INFINITY)-b); if (u>maxulp_small) maxulp_small=u; }
    }
    printf("max rel %.3e at x=%.6f ; max ulp for x>-5: %.2f\n", maxrel, worstx, maxulp_small);
}
