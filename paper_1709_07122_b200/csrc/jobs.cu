// jobs.cu -- the job runtime of include/pcpm.h (pcpm_runtime_*, pcpm_job_*): whole
// PageRank jobs from HOST memory (the e2e path of bench.py), pipelined natively.
//
// A job = host CSR -> H2D copy -> layout build (a0) -> `iters` PageRank iterations
// (a1-a4) -> D2H of PR.  One worker thread runs the jobs in submission order on a
// compute stream; a copy stream uploads job k+1's CSR while job k builds and
// iterates, and a third stream brings job k-1's result back, so the PCIe copy
// engines and the SMs stay busy at once (the GPU analogue of the paper's running
// PageRank on one graph after another).  Only one layout is resident: job
// k-1's handle is destroyed before job k is built.
#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <thread>

#include "pcpm_internal.cuh"

namespace pcpm {
namespace {

struct Job {
  int64_t id = 0;
  pcpm_csr csr{};          // host (or device) arrays, borrowed until the job completes
  int bits = 0;
  unsigned flags = 0;
  double d = 0.85;
  int iters = 0;
  float* out = nullptr;    // n floats, host or device
  // device state
  int64_t* rp = nullptr;
  uint32_t* col = nullptr;
  float* val = nullptr;
  float* dout = nullptr;
  cudaEvent_t uploaded = nullptr, done = nullptr;
  bool upload_issued = false;
  int status = 0;          // PCPM_* of the job
  std::string msg;
  bool finished = false;
};

}  // namespace
}  // namespace pcpm

struct pcpm_runtime {
  int device = 0;
  cudaStream_t comp = nullptr, up = nullptr, down = nullptr;
  std::thread worker;
  std::mutex mu;
  std::condition_variable cv;           // queue changes / job completion
  std::deque<pcpm::Job*> queue;         // submitted, not yet run
  std::map<int64_t, pcpm::Job*> jobs;   // every job not yet waited for
  int64_t next_id = 1;
  bool stop = false;
};

namespace pcpm {
namespace {

// H2D of the job's CSR on the copy stream (device arrays from the stream-ordered pool)
int issue_upload(pcpm_runtime* rt, Job* j) {
  const int64_t n = j->csr.n_src, m = j->csr.nnz;
  cudaStream_t s = rt->up;
  auto dev = [](const void* p) { return is_device_ptr(p); };
  if (!dev(j->csr.row_ptr)) {
    PCPM_CK(cudaMallocAsync(reinterpret_cast<void**>(&j->rp), sizeof(int64_t) * (n + 1), s));
    PCPM_CK(cudaMemcpyAsync(j->rp, j->csr.row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  }
  if (m > 0 && !dev(j->csr.col_idx)) {
    PCPM_CK(cudaMallocAsync(reinterpret_cast<void**>(&j->col), sizeof(uint32_t) * m, s));
    PCPM_CK(cudaMemcpyAsync(j->col, j->csr.col_idx, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, s));
  }
  if (m > 0 && j->csr.values && !dev(j->csr.values)) {
    PCPM_CK(cudaMallocAsync(reinterpret_cast<void**>(&j->val), sizeof(float) * m, s));
    PCPM_CK(cudaMemcpyAsync(j->val, j->csr.values, sizeof(float) * m, cudaMemcpyHostToDevice, s));
  }
  PCPM_CK(cudaEventRecord(j->uploaded, s));
  j->upload_issued = true;
  return PCPM_OK;
}

void finish(pcpm_runtime* rt, Job* j, int status, const std::string& msg) {
  std::lock_guard<std::mutex> lk(rt->mu);
  j->status = status;
  j->msg = msg;
  j->finished = true;
  rt->cv.notify_all();
}

// Build + iterate one job (worker thread); `prev` is the previous job's handle, destroyed
// here once this job's upload is in flight (it synchronises the compute stream).
int run_job(pcpm_runtime* rt, Job* j, pcpm_handle** prev, Job* next) {
  int rc;
  if (!j->upload_issued && (rc = issue_upload(rt, j))) return rc;
  // the next job's CSR starts uploading now, under this job's build and iterations
  if (next && !next->upload_issued && (rc = issue_upload(rt, next))) return rc;
  if (*prev) {
    pcpm_destroy(*prev);
    *prev = nullptr;
  }
  PCPM_CK(cudaStreamWaitEvent(rt->comp, j->uploaded, 0));
  pcpm_csr c = j->csr;
  if (j->rp) c.row_ptr = j->rp;
  if (j->col) c.col_idx = j->col;
  if (j->val) c.values = j->val;
  pcpm_handle* h = pcpm_build_ex(&c, j->bits, j->flags, rt->comp);
  if (!h) return pcpm_last_status() ? pcpm_last_status() : PCPM_ECUDA;
  // the device CSR copies are no longer needed once the layout exists
  if (j->rp) PCPM_CK(cudaFreeAsync(j->rp, rt->comp));
  if (j->col) PCPM_CK(cudaFreeAsync(j->col, rt->comp));
  if (j->val) PCPM_CK(cudaFreeAsync(j->val, rt->comp));
  j->rp = nullptr;
  j->col = nullptr;
  j->val = nullptr;
  *prev = h;
  if (j->csr.values && (j->flags & PCPM_KEEP_VALUES)) {
    if ((rc = pcpm_set_option(h, "weighted_pagerank", 1))) return rc;
  }
  const bool dev_out = is_device_ptr(j->out);
  float* dst = j->out;
  if (!dev_out) {
    PCPM_CK(cudaMallocAsync(reinterpret_cast<void**>(&j->dout), sizeof(float) * j->csr.n_src, rt->comp));
    dst = j->dout;
  }
  if ((rc = pcpm_pagerank(h, j->d, j->iters, dst))) return rc;
  if (!dev_out) {
    cudaEvent_t it_done;
    PCPM_CK(cudaEventCreateWithFlags(&it_done, cudaEventDisableTiming));
    PCPM_CK(cudaEventRecord(it_done, rt->comp));
    PCPM_CK(cudaStreamWaitEvent(rt->down, it_done, 0));
    PCPM_CK(cudaEventDestroy(it_done));
    PCPM_CK(cudaMemcpyAsync(j->out, j->dout, sizeof(float) * j->csr.n_src, cudaMemcpyDeviceToHost, rt->down));
    PCPM_CK(cudaFreeAsync(j->dout, rt->down));
    j->dout = nullptr;
    PCPM_CK(cudaEventRecord(j->done, rt->down));
  } else {
    PCPM_CK(cudaEventRecord(j->done, rt->comp));
  }
  return PCPM_OK;
}

void worker_main(pcpm_runtime* rt) {
  cudaSetDevice(rt->device);
  pcpm_handle* prev = nullptr;
  for (;;) {
    Job* j = nullptr;
    Job* next = nullptr;
    {
      std::unique_lock<std::mutex> lk(rt->mu);
      rt->cv.wait(lk, [&] { return rt->stop || !rt->queue.empty(); });
      if (rt->queue.empty()) break;             // stop requested and nothing left
      j = rt->queue.front();
      rt->queue.pop_front();
      if (!rt->queue.empty()) next = rt->queue.front();
    }
    set_error(PCPM_OK, "");
    const int rc = run_job(rt, j, &prev, next);
    std::string msg;
    if (rc) {
      char buf[512];
      pcpm_last_error(buf, sizeof(buf));
      msg = buf;
      // leave the streams usable for the next job
      cudaStreamSynchronize(rt->comp);
      cudaStreamSynchronize(rt->up);
      cudaGetLastError();
      if (j->rp) cudaFree(j->rp);
      if (j->col) cudaFree(j->col);
      if (j->val) cudaFree(j->val);
      j->rp = nullptr;
      j->col = nullptr;
      j->val = nullptr;
    }
    finish(rt, j, rc, msg);
  }
  if (prev) pcpm_destroy(prev);
}

}  // namespace
}  // namespace pcpm

using namespace pcpm;

extern "C" {

pcpm_runtime* pcpm_runtime_create(void) {
  set_error(PCPM_OK, "");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_error(PCPM_ECUDA, "no CUDA device");
    return nullptr;
  }
  pcpm_runtime* rt = new pcpm_runtime();
  cudaGetDevice(&rt->device);
  if (cudaStreamCreateWithFlags(&rt->comp, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&rt->up, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&rt->down, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    set_error(PCPM_ECUDA, "stream creation failed");
    if (rt->comp) cudaStreamDestroy(rt->comp);
    if (rt->up) cudaStreamDestroy(rt->up);
    if (rt->down) cudaStreamDestroy(rt->down);
    delete rt;
    return nullptr;
  }
  rt->worker = std::thread(worker_main, rt);
  return rt;
}

int pcpm_job_submit(pcpm_runtime* rt, const pcpm_csr* csr, int partition_bits, unsigned flags, double d, int iters,
                    float* out, int64_t* job_id) {
  if (!rt || !csr || !csr->row_ptr || (csr->nnz > 0 && !csr->col_idx) || !out || !job_id) {
    set_error(PCPM_EINVAL, "NULL runtime, csr, output or job id");
    return PCPM_EINVAL;
  }
  if (!(d > 0.0 && d < 1.0) || iters < 0 || csr->n_src != csr->n_dst || csr->n_src < 1) {
    set_error(PCPM_EINVAL, "d must be in (0,1), iters >= 0 and the graph square (PageRank jobs)");
    return PCPM_EINVAL;
  }
  Job* j = new Job();
  j->csr = *csr;
  j->bits = partition_bits;
  j->flags = flags;
  j->d = d;
  j->iters = iters;
  j->out = out;
  if (cudaEventCreateWithFlags(&j->uploaded, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&j->done, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    if (j->uploaded) cudaEventDestroy(j->uploaded);
    delete j;
    set_error(PCPM_ECUDA, "event creation failed");
    return PCPM_ECUDA;
  }
  {
    std::lock_guard<std::mutex> lk(rt->mu);
    j->id = rt->next_id++;
    rt->jobs[j->id] = j;
    rt->queue.push_back(j);
  }
  rt->cv.notify_all();
  *job_id = j->id;
  return PCPM_OK;
}

int pcpm_job_wait(pcpm_runtime* rt, int64_t job_id) {
  if (!rt) {
    set_error(PCPM_EINVAL, "NULL runtime");
    return PCPM_EINVAL;
  }
  Job* j = nullptr;
  {
    std::unique_lock<std::mutex> lk(rt->mu);
    auto it = rt->jobs.find(job_id);
    if (it == rt->jobs.end()) {
      set_error(PCPM_EINVAL, "unknown (or already waited-for) job id");
      return PCPM_EINVAL;
    }
    j = it->second;
    rt->cv.wait(lk, [&] { return j->finished; });
    rt->jobs.erase(it);
  }
  int rc = j->status;
  std::string msg = j->msg;
  if (rc == PCPM_OK && cudaEventSynchronize(j->done) != cudaSuccess) {
    rc = PCPM_ECUDA;
    msg = std::string("job failed on the device: ") + cudaGetErrorString(cudaGetLastError());
  }
  cudaEventDestroy(j->uploaded);
  cudaEventDestroy(j->done);
  delete j;
  if (rc) set_error(rc, msg);
  return rc;
}

void pcpm_runtime_destroy(pcpm_runtime* rt) {
  if (!rt) return;
  {
    std::lock_guard<std::mutex> lk(rt->mu);
    rt->stop = true;
  }
  rt->cv.notify_all();
  if (rt->worker.joinable()) rt->worker.join();
  cudaStreamSynchronize(rt->comp);
  cudaStreamSynchronize(rt->up);
  cudaStreamSynchronize(rt->down);
  for (auto& kv : rt->jobs) {                   // submitted but never waited for
    cudaEventDestroy(kv.second->uploaded);
    cudaEventDestroy(kv.second->done);
    delete kv.second;
  }
  cudaStreamDestroy(rt->comp);
  cudaStreamDestroy(rt->up);
  cudaStreamDestroy(rt->down);
  delete rt;
}

}  // extern "C"
