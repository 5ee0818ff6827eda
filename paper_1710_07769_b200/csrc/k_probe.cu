// k_probe.cu -- gather-only probe of the numeric pass (measurement, SURVEY.md
// §8(d) D3 / north star: "L2 hit rate on the A^T gathers").  ncu cannot
// attribute a hit rate to one array inside the numeric kernels, so this
// kernel runs the same gather loop -- rows in ascending order, warp per row,
// for each entry k of row i the column k of the CSC of A_hat (rows and
// values, 32 lanes per step) -- with no accumulation, no sort and no writes
// except one checksum per warp (so the loads cannot be elided).  Its L2 and
// DRAM counters are the gathers' own.
#include "common.cuh"

namespace rig {

constexpr int kProbeThreads = 256;

__global__ void __launch_bounds__(kProbeThreads) k_gather_probe(Csr A, Csc T, int64_t rb, int64_t re, double *sink) {
    const int l = lane_id();
    const int64_t nw = ((int64_t)gridDim.x * kProbeThreads) >> 5;
    double acc = 0.0;
    int jx = 0;
    for (int64_t i = rb + (((int64_t)blockIdx.x * kProbeThreads + threadIdx.x) >> 5); i < re; i += nw) {
        const int64_t s = A.rp[i], e = A.rp[i + 1];
        for (int64_t bb = s; bb < e; bb += 32) {
            const int nent = (int)min((int64_t)32, e - bb);
            int64_t cs = 0;
            int cl = 0;
            if (l < nent) {
                const int k = A.ci[bb + l];
                const int64_t c0 = T.cp[k];
                cl = (int)(T.cp[k + 1] - c0);
                cs = c0 + k;
            }
            for (int t = 0; t < nent; ++t) {
                const int64_t q0 = __shfl_sync(kFull, cs, t);
                const int len = __shfl_sync(kFull, cl, t);
                for (int off = l; off < len; off += 32) {
                    jx ^= __ldg(&T.ri[q0 + off]);
                    acc += __ldg(&T.vt[q0 + off]);
                }
            }
        }
    }
    acc += (double)jx;
    acc = warp_sum(acc);
    if (l == 0) sink[((int64_t)blockIdx.x * kProbeThreads + threadIdx.x) >> 5] = acc;
}

int gather_probe_warps() { return num_sms() * 16 * (kProbeThreads / 32); }

void launch_gather_probe(const Csr &A, const Csc &T, int64_t rb, int64_t re, double *sink, cudaStream_t s) {
    k_gather_probe<<<num_sms() * 16, kProbeThreads, 0, s>>>(A, T, rb, re, sink);
    note_launch();
}

}  // namespace rig
