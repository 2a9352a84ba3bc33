// comm.cu — the gradient exchange of the sample-sharded step and
// its failure handling.
//
//   * One SUM-allreduce of [acc_μ | acc_ρ | L_data] over all K·G ranks ("the
//     gradients are averaged across all GPUs", Alg. 2 l.13-15 P:263-264). The global 1/(S·B)
//     pre-scaling makes the sum exact for every grid (R8).
//   * Layer-bucketed on a dedicated comm stream (ResNet path): while the backward still runs
//     on the compute streams, each bucket of layers whose acc_μ / acc_ρ segments are final
//     (their wgrad, ε combine and bias kernels have run in the last sample chunk) is reduced —
//     stage-4 layers (≈ 75 % of the bytes) finish first, so most of the 89 MB moves behind the
//     remaining stages' backward. The tail bucket (first layers + L_data) follows the backward;
//     the compute stream waits for the comm stream only before the finalize reads acc.
//   * Non-blocking communicator with a timeout ("fail loudly", S:733 exit code 3): init,
//     every NCCL call and every host sync poll ncclCommGetAsyncError; an error or a peer that
//     does not answer within comm_timeout_ms aborts the communicator (ncclCommAbort) and the
//     call returns BNN_ERR_COMM. The context is unusable afterwards (bnn_destroy only).
#include <chrono>
#include <cstdlib>
#include <thread>

#include "ctx.cuh"

namespace {
double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int comm_fail(bnn_ctx* c, const char* what, const char* why) {
    if (c->comm && !c->comm_aborted) {
        ncclCommAbort(c->comm);
        c->comm_aborted = true;
    }
    c->comm = nullptr;
    return c->set_err(BNN_ERR_COMM, "%s: %s (communicator aborted)", what, why);
}
}  // namespace

// Wait for a non-blocking NCCL call (or the communicator's init) to leave ncclInProgress.
int comm_check(bnn_ctx* c, ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress) return comm_fail(c, what, ncclGetErrorString(r));
    const double t0 = now_ms();
    while (r == ncclInProgress) {
        ncclResult_t st = ncclSuccess;
        ncclResult_t q = ncclCommGetAsyncError(c->comm, &st);
        if (q != ncclSuccess) return comm_fail(c, what, ncclGetErrorString(q));
        if (st == ncclSuccess) break;
        if (st != ncclInProgress) return comm_fail(c, what, ncclGetErrorString(st));
        if (now_ms() - t0 > c->comm_timeout_ms) return comm_fail(c, what, "timeout (a peer did not answer)");
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    return BNN_OK;
}

int comm_init(bnn_ctx* c, const uint8_t* uid, int world, int rank) {
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;  // every call returns at once; completion and errors are polled
    ncclResult_t r = ncclCommInitRankConfig(&c->comm, world, id, rank, &cfg);
    if (r != ncclSuccess && r != ncclInProgress) {
        c->comm = nullptr;
        return c->set_err(BNN_ERR_COMM, "ncclCommInitRankConfig: %s", ncclGetErrorString(r));
    }
    int rc = comm_check(c, ncclInProgress, "ncclCommInitRankConfig");
    if (rc) return rc;
    if (cudaStreamCreateWithFlags(&c->comm_st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_comm_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_comm_out, cudaEventDisableTiming) != cudaSuccess)
        return c->set_err(BNN_ERR_CUDA, "comm stream creation failed");
    const char* e = getenv("BNN_AR_BUCKET_MB");
    c->ar_bucket_bytes = (int64_t)((e ? atof(e) : 16.0) * (1 << 20));
    return BNN_OK;
}

// Host wait for everything enqueued on `st` (and the comm stream), checking the communicator
// while waiting: a failed or silent peer turns into BNN_ERR_COMM instead of a hang.
int comm_sync(bnn_ctx* c, cudaStream_t st) {
    if (!c->comm) {
        if (c->comm_aborted) return c->set_err(BNN_ERR_COMM, "communicator was aborted by an earlier error");
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return c->set_err(BNN_ERR_CUDA, "cudaStreamSynchronize: %s", cudaGetErrorString(e));
        return BNN_OK;
    }
    const double t0 = now_ms();
    for (cudaStream_t q : {c->comm_st, st}) {
        for (;;) {
            cudaError_t e = cudaStreamQuery(q);
            if (e == cudaSuccess) break;
            if (e != cudaErrorNotReady) return c->set_err(BNN_ERR_CUDA, "cudaStreamQuery: %s", cudaGetErrorString(e));
            ncclResult_t as = ncclSuccess;
            ncclResult_t r = ncclCommGetAsyncError(c->comm, &as);
            if (r != ncclSuccess) return comm_fail(c, "ncclCommGetAsyncError", ncclGetErrorString(r));
            if (as != ncclSuccess && as != ncclInProgress) return comm_fail(c, "collective", ncclGetErrorString(as));
            if (now_ms() - t0 > c->comm_timeout_ms) return comm_fail(c, "step", "timeout (a collective did not complete)");
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
    return BNN_OK;
}

// ---------------------------------------------------------------- bucketed allreduce
void ar_begin(bnn_ctx* c) {
    const int L = (int)c->layers.size();
    c->ar_done.assign(L, 0);
    c->ar_top = L - 1;
    c->ar_buckets = 0;
    if (c->ar_ev.size() != (size_t)L) {
        for (auto& p : c->ar_ev)
            for (cudaEvent_t e : p)
                if (e) cudaEventDestroy(e);
        c->ar_ev.assign(L, {nullptr, nullptr});
        for (auto& p : c->ar_ev)
            for (cudaEvent_t& e : p) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
}

namespace {
// one bucket: params [off_lo, off_hi) of acc_μ and acc_ρ (+ L_data when `with_loss`), on the
// comm stream, in one NCCL group
int ar_issue(bnn_ctx* c, int64_t off_lo, int64_t off_hi, bool with_loss) {
    float* acc = c->acc;
    const size_t n = (size_t)(off_hi - off_lo);
    int rc = comm_check(c, ncclGroupStart(), "ncclGroupStart");
    if (rc) return rc;
    if (n) {
        rc = comm_check(c, ncclAllReduce(acc + off_lo, acc + off_lo, n, ncclFloat32, ncclSum, c->comm, c->comm_st),
                        "ncclAllReduce(acc_mu bucket)");
        if (rc) return rc;
        rc = comm_check(c, ncclAllReduce(acc + c->P_pad + off_lo, acc + c->P_pad + off_lo, n, ncclFloat32, ncclSum,
                                         c->comm, c->comm_st),
                        "ncclAllReduce(acc_rho bucket)");
        if (rc) return rc;
    }
    if (with_loss) {
        rc = comm_check(c, ncclAllReduce(acc + 2 * c->P_pad, acc + 2 * c->P_pad, 1, ncclFloat32, ncclSum, c->comm,
                                         c->comm_st),
                        "ncclAllReduce(L_data)");
        if (rc) return rc;
    }
    rc = comm_check(c, ncclGroupEnd(), "ncclGroupEnd");
    if (rc) return rc;
    ++c->ar_buckets;
    return BNN_OK;
}

int64_t layer_lo(const bnn_ctx* c, int l) { return c->layers[l].off_w; }
int64_t layer_hi(const bnn_ctx* c, int l) { return c->layers[l].off_b + c->layers[l].cout; }
}  // namespace

// Layer l's acc segments are final once the work already enqueued on `w0` / `w1` completes.
// Reduce every complete run of layers [lo, top] (top = the highest not yet reduced) that has
// reached the bucket size.
int ar_layer_done(bnn_ctx* c, int l, cudaStream_t w0, cudaStream_t w1) {
    if (!c->ar_live) return BNN_OK;
    cudaEventRecord(c->ar_ev[l][0], w0);
    cudaEventRecord(c->ar_ev[l][1], w1);
    c->ar_done[l] = 1;
    int lo = c->ar_top + 1;
    while (lo > 0 && c->ar_done[lo - 1]) --lo;
    if (lo > c->ar_top) return BNN_OK;
    const int64_t bytes = 8 * (layer_hi(c, c->ar_top) - layer_lo(c, lo));
    if (bytes < c->ar_bucket_bytes || lo == 0) return BNN_OK;  // layer 0's bucket carries L_data: at the end
    for (int k = lo; k <= c->ar_top; ++k)
        for (cudaEvent_t e : c->ar_ev[k]) cudaStreamWaitEvent(c->comm_st, e, 0);
    int rc = ar_issue(c, layer_lo(c, lo), layer_hi(c, c->ar_top), false);
    c->ar_top = lo - 1;
    return rc;
}

// After the backward: the remaining layers [0, top] and L_data (everything on `st` is then
// final), and the compute stream waits for the comm stream before the finalize reads acc.
int ar_finish(bnn_ctx* c, cudaStream_t st) {
    cudaEventRecord(c->ev_comm_in, st);
    cudaStreamWaitEvent(c->comm_st, c->ev_comm_in, 0);
    int rc;
    if (c->ar_top >= 0)
        rc = ar_issue(c, 0, c->ar_live_used ? layer_hi(c, c->ar_top) : c->P_pad, true);
    else
        rc = ar_issue(c, 0, 0, true);
    if (rc) return rc;
    cudaEventRecord(c->ev_comm_out, c->comm_st);
    cudaStreamWaitEvent(st, c->ev_comm_out, 0);
    return BNN_OK;
}

void comm_destroy(bnn_ctx* c) {
    if (c->comm) {
        if (c->comm_st) cudaStreamSynchronize(c->comm_st);
        ncclCommFinalize(c->comm);
        comm_check(c, ncclInProgress, "ncclCommFinalize");
        if (c->comm) ncclCommDestroy(c->comm);
        c->comm = nullptr;
    }
    if (c->comm_st) cudaStreamDestroy(c->comm_st);
    for (cudaEvent_t e : {c->ev_comm_in, c->ev_comm_out})
        if (e) cudaEventDestroy(e);
    for (auto& p : c->ar_ev)
        for (cudaEvent_t e : p)
            if (e) cudaEventDestroy(e);
}

