// Host-side helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <string>

// records the message returned by pdf_last_error() and returns `code`
int pdf_fail(int code, const std::string& msg);

#define PDF_CK(expr)                                                                        \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) return pdf_fail(PDF_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct pdf_ctx;
// grid edge M and element type (enum pdf_dtype) of a context
int pdf_ctx_info(const pdf_ctx* c, int* M, int* dtype);
