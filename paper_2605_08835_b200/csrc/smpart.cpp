// SM partitioning of UNet ∥ VAE with CUDA green contexts (the contention mechanism of
// PAPER.md:146-148 §II-C and :262): two green contexts on disjoint SM sets, one stream each. A kernel
// launched on a partition stream runs only on that partition's SMs, so the persistent kernels size their
// grids by stream_sms(stream) (the partition's SM count) instead of the whole chip's.
#include <cuda.h>

#include <mutex>
#include <stdexcept>
#include <unordered_map>

#include "api_common.h"
#include "common.cuh"
#include "kernels.h"

namespace sd {

namespace {
struct Drv {
  CUresult (*devGetRes)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*split)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                    unsigned int) = nullptr;
  CUresult (*genDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int) = nullptr;
  CUresult (*gcCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
  CUresult (*gcDestroy)(CUgreenCtx) = nullptr;
  CUresult (*gcStream)(CUstream*, CUgreenCtx, unsigned int, int) = nullptr;
  CUresult (*devGet)(CUdevice*, int) = nullptr;
  bool ok = false;
};

template <class F>
void sym(const char* name, F* f) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    *f = reinterpret_cast<F>(p);
}

Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    sym("cuDeviceGetDevResource", &d.devGetRes);
    sym("cuDevSmResourceSplitByCount", &d.split);
    sym("cuDevResourceGenerateDesc", &d.genDesc);
    sym("cuGreenCtxCreate", &d.gcCreate);
    sym("cuGreenCtxDestroy", &d.gcDestroy);
    sym("cuGreenCtxStreamCreate", &d.gcStream);
    sym("cuDeviceGet", &d.devGet);
    d.ok = d.devGetRes && d.split && d.genDesc && d.gcCreate && d.gcDestroy && d.gcStream && d.devGet;
  });
  return d;
}

std::mutex g_mu;
std::unordered_map<cudaStream_t, int> g_stream_sms;  // partition streams → their SM count

void check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw CudaError(std::string(what) + " failed: CUresult " + std::to_string((int)r));
}
}  // namespace

int stream_sms(cudaStream_t st) {
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_stream_sms.find(st);
    if (it != g_stream_sms.end()) return it->second;
  }
  return num_sms();
}

struct Partition {
  CUgreenCtx gc[2] = {nullptr, nullptr};
  cudaStream_t st[2] = {nullptr, nullptr};
  int sms[2] = {0, 0};
};

// group 0 = the VAE partition (vae_sms SMs, rounded up by the driver to its granularity: 8 on sm_90+),
// group 1 = the remaining SMs (the UNet); stream priorities as in the non-partitioned server
Partition* partition_create(int device, int vae_sms) {
  Drv& d = drv();
  if (!d.ok) throw std::runtime_error("green contexts unavailable in this driver");
  CUdevice dev;
  check(d.devGet(&dev, device), "cuDeviceGet");
  CUdevResource all{};
  check(d.devGetRes(dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
  CUdevResource grp{}, rest{};
  unsigned int n = 1;
  check(d.split(&grp, &n, &all, &rest, 0, (unsigned)vae_sms), "cuDevSmResourceSplitByCount");
  if (n != 1) throw std::runtime_error("SM split produced no group");
  auto* p = new Partition();
  CUdevResource res[2] = {grp, rest};
  int lo_p, hi_p;
  SD_CUDA(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
  for (int i = 0; i < 2; ++i) {
    CUdevResourceDesc desc;
    check(d.genDesc(&desc, &res[i], 1), "cuDevResourceGenerateDesc");
    check(d.gcCreate(&p->gc[i], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
    CUstream s;
    check(d.gcStream(&s, p->gc[i], CU_STREAM_NON_BLOCKING, i == 0 ? lo_p : hi_p), "cuGreenCtxStreamCreate");
    p->st[i] = reinterpret_cast<cudaStream_t>(s);
    p->sms[i] = (int)res[i].sm.smCount;
  }
  std::lock_guard<std::mutex> g(g_mu);
  for (int i = 0; i < 2; ++i) g_stream_sms[p->st[i]] = p->sms[i];
  return p;
}

cudaStream_t partition_stream(Partition* p, int i) { return p->st[i]; }

void partition_destroy(Partition* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> g(g_mu);
    for (int i = 0; i < 2; ++i) g_stream_sms.erase(p->st[i]);
  }
  for (int i = 0; i < 2; ++i) {
    if (p->st[i]) cudaStreamDestroy(p->st[i]);
    if (p->gc[i]) drv().gcDestroy(p->gc[i]);
  }
  delete p;
}

}  // namespace sd

struct sd_partition {
  sd::Partition* p;
};

extern "C" sd_status sd_sm_partition_create(int32_t device, int32_t vae_sms, sd_partition** out, void** unet_stream,
                                            void** vae_stream, int32_t* unet_sms, int32_t* vae_sms_out) {
  SD_REQUIRE(out && unet_stream && vae_stream && vae_sms >= 1, "sd_sm_partition_create: bad args");
  SD_API_BEGIN
  SD_CUDA(cudaSetDevice(device));
  SD_CUDA(cudaFree(nullptr));  // primary context current
  auto* h = new sd_partition{sd::partition_create(device, vae_sms)};
  *unet_stream = h->p->st[1];
  *vae_stream = h->p->st[0];
  if (unet_sms) *unet_sms = h->p->sms[1];
  if (vae_sms_out) *vae_sms_out = h->p->sms[0];
  *out = h;
  SD_API_END
}

extern "C" sd_status sd_sm_partition_destroy(sd_partition* h) {
  if (!h) return SD_OK;
  sd::partition_destroy(h->p);
  delete h;
  return SD_OK;
}
