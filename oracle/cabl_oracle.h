/* TEST INFRASTRUCTURE ONLY — CPU oracle for the DOT / GEMV / GER path.
 * See cabl_oracle.c for the reference citations and FP semantics. */
#ifndef CABL_ORACLE_H
#define CABL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t oracle_sm64_key(uint64_t seed, uint64_t stream);
uint64_t oracle_sm64(uint64_t key, uint64_t index);
void oracle_gen_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t stream,
                            uint64_t offset);
void oracle_gen_uniform_f64(double* out, uint64_t n, uint64_t seed, uint64_t stream,
                            uint64_t offset);
void oracle_gen_normal_f64(double* out, uint64_t n, uint64_t seed, uint64_t stream,
                           uint64_t offset);

float oracle_dot_ref_f32(const float* x, const float* y, uint64_t n, float alpha0,
                         unsigned vec);
double oracle_dot_ref_f64(const double* x, const double* y, uint64_t n, double alpha0,
                          unsigned vec);
void oracle_gemv_ref_f32(const float* A, int layout, uint64_t m, uint64_t n, const float* x,
                         float* c, unsigned vec);
void oracle_gemv_ref_f64(const double* A, int layout, uint64_t m, uint64_t n,
                         const double* x, double* c, unsigned vec);
void oracle_ger_ref_f32(const float* x, const float* y, float* C, int layout, uint64_t m,
                        uint64_t n);
void oracle_ger_ref_f64(const double* x, const double* y, double* C, int layout, uint64_t m,
                        uint64_t n);

void oracle_dot_truth_f32(const float* x, const float* y, uint64_t n, float alpha0,
                          double* truth, double* sumabs);
void oracle_dot_truth_f64(const double* x, const double* y, uint64_t n, double alpha0,
                          double* truth, double* sumabs);
void oracle_gemv_truth_f32(const float* A, int layout, uint64_t m, uint64_t n, const float* x,
                           const float* c0, double* truth, double* rowabs);
void oracle_gemv_truth_f64(const double* A, int layout, uint64_t m, uint64_t n,
                           const double* x, const double* c0, double* truth, double* rowabs);

#ifdef __cplusplus
}
#endif

#endif
