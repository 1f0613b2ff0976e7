// launch bookkeeping shared by the kernel translation units
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cml {
int check_launch(const char* what);   // cudaGetLastError + launch counter
void count_launch();
void set_error(const char* msg);
int num_sms();
}  // namespace cml
