// Internal declarations of libbf.so (not part of the public ABI).
#pragma once

#include "../../include/bf.h"

#define BF_MAX_RADIUS 1024

struct bf_plan {
  int ks, kr;
  double sigma_s, sigma_r;
  int radius, n_terms;
  double D;
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
};
