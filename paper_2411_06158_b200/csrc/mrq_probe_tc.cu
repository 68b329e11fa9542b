// mrq_probe_tc.cu -- tcgen05 tensor-core probe screen (placeholder until the
// UMMA kernel lands: the CUDA-core fp32 screen in mrq_kernels.cu is used).
#include "mrq_probe_tc.cuh"

int mrq_probe_tc_init(mrq_index *) { return MRQ_OK; }
void mrq_probe_tc_free(mrq_index *) {}
bool mrq_probe_tc_enabled(const mrq_index *) { return false; }
double mrq_probe_tc_kappa(const mrq_index *) { return 0.0; }
int mrq_probe_tc_run(mrq_index *, const float *, int64_t, float *, cudaStream_t)
{
    mrq_set_error("tcgen05 probe not available");
    return MRQ_ECUDA;
}
