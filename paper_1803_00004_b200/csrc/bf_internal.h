// Internal declarations of libbf.so (not part of the public ABI).
#pragma once

#include "../../include/bf.h"

#define BF_MAX_RADIUS 1024
#define BF_MAX_SP_PASSES 32

struct bf_plan {
  int ks, kr;
  double sigma_s, sigma_r;
  int radius, n_terms;
  double D;
  double T;        // period half-width of the cosine basis: D, or T_r for the literal window
  int literal;     // BF_RANGE_WINDOW_LITERAL
  int input_dtype;
  bf_plan_options opt;
  // range plan Lambda^r: selected k ascending and a_k
  int n_k;
  int k[BF_MAX_TERMS];
  double a[BF_MAX_TERMS];
  // spatial plan Lambda^s
  int n_sp;
  int sp_family[BF_MAX_SPATIAL_TERMS];
  int sp_j1[BF_MAX_SPATIAL_TERMS], sp_k1[BF_MAX_SPATIAL_TERMS];
  int sp_j2[BF_MAX_SPATIAL_TERMS], sp_k2[BF_MAX_SPATIAL_TERMS];
  double sp_coef[BF_MAX_SPATIAL_TERMS];
  // separable factorisation K~_s(u, v) = fx(u) fy(v), each a sum of boxes w [lo, hi]
  int separable;
  int nbx, nby;
  int lox[BF_MAX_AXIS_BOXES], hix[BF_MAX_AXIS_BOXES];
  double wx[BF_MAX_AXIS_BOXES];
  int loy[BF_MAX_AXIS_BOXES], hiy[BF_MAX_AXIS_BOXES];
  double wy[BF_MAX_AXIS_BOXES];
  // box-pair form for the GPU path (NEXT f3): K~_s(v, u) = sum_{s < ns} fx_s(u) fy_s(v), each
  // factor a sum of boxes. ns = 1 is the separable plan above; ns = 2 covers the rank-2 plans
  // (N_s = 5, the paper's three boxes), with fx_s = one nested elementary box each.
  int ns;
  int snbx[2], slox[2][BF_MAX_AXIS_BOXES], shix[2][BF_MAX_AXIS_BOXES];
  double swx[2][BF_MAX_AXIS_BOXES];
  int snby[2], sloy[2][BF_MAX_AXIS_BOXES], shiy[2][BF_MAX_AXIS_BOXES];
  double swy[2][BF_MAX_AXIS_BOXES];
  // general plans (NEXT f3: no separable / rank-2 form, e.g. N_s = 13, 25 at J = 4): K~_s as a sum
  // of n_pass separable box products (an exact rank factorisation of the kernel's box-weight matrix,
  // each factor's boxes cut into groups of at most BF_MAX_AXIS_BOXES); the GPU runs one separable
  // pass per product and accumulates num / den in fp64 (ns = 0 then).
  int n_pass;
  int rank;
  struct {
    int nbx, nby;
    int lox[BF_MAX_AXIS_BOXES], hix[BF_MAX_AXIS_BOXES];
    double wx[BF_MAX_AXIS_BOXES];
    int loy[BF_MAX_AXIS_BOXES], hiy[BF_MAX_AXIS_BOXES];
    double wy[BF_MAX_AXIS_BOXES];
  } pass[BF_MAX_SP_PASSES];
};
