// The allreduce hook of the term-sharded Kronecker operator (kb_forward.allreduce) as a
// C function over NCCL: ncclAllReduce(sum, fp64) on the communicator torch's
// ProcessGroupNCCL owns (passed as the hook's context), stream-ordered on the
// solve's stream -- no Python callback inside kb_cgls_run / kb_sb_run.  The NCCL
// library is the one torch already loaded (dlopen RTLD_NOLOAD of libnccl.so.2), so
// the communicator pointer is valid for it.
#include <dlfcn.h>

#include <atomic>

#include "kb_common.cuh"

namespace {
// ncclResult_t ncclAllReduce(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t)
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
constexpr int NCCL_FLOAT64 = 8, NCCL_SUM = 0;   // nccl.h enum values
nccl_allreduce_t g_allreduce = nullptr;
std::atomic<int> g_nccl_error{0};

bool resolve() {
    if (g_allreduce) return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return false;
    g_allreduce = reinterpret_cast<nccl_allreduce_t>(dlsym(h, "ncclAllReduce"));
    return g_allreduce != nullptr;
}
}  // namespace

extern "C" void kb_nccl_allreduce_f64(void* comm, double* buf, int64_t count, kb_stream_t stream) {
    if (!resolve()) {
        g_nccl_error = -1;
        return;
    }
    const int rc = g_allreduce(buf, buf, (size_t)count, NCCL_FLOAT64, NCCL_SUM, comm, kb::as_stream(stream));
    if (rc != 0) g_nccl_error = rc;
}

extern "C" int kb_nccl_available(void) { return resolve() ? 1 : 0; }

extern "C" int kb_nccl_last_error(int reset) {
    const int e = g_nccl_error.load();
    if (reset) g_nccl_error = 0;
    return e;
}
