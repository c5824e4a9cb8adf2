// dsi_collective.cpp -- the one exchange step of the path: NCCL loaded with
// dlopen (reusing torch's libnccl when mapped), the grouped all-reduce of the per-config
// integer moments, and -- test build only -- the host all-reduce hook and A/B knobs.
#include "dsi_host.h"

using namespace dsih;
#include <dlfcn.h>

namespace dsih {

NcclApi &nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // Reuse a libnccl already mapped into the process (e.g. torch's), else load one.
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.lib = h;
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
      api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.CommCount = (decltype(api.CommCount))dlsym(h, "ncclCommCount");
      api.CommUserRank = (decltype(api.CommUserRank))dlsym(h, "ncclCommUserRank");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
               api.GroupStart && api.GroupEnd && api.GetErrorString;
    }
  }
  return api;
}

namespace {
// Test hook (dsi_set_host_allreduce): cross-rank sums through a caller-supplied host function
// instead of NCCL, so multi-rank runs can be exercised where NCCL cannot form a communicator
// (several ranks on one GPU).
dsi_host_allreduce_fn g_host_ar = nullptr;
void *g_host_ar_user = nullptr;
}  // namespace

bool host_hook_set() { return g_host_ar != nullptr; }
bool host_hook_sum(uint64_t *buf, size_t count) { return g_host_ar && g_host_ar(buf, count, g_host_ar_user) == 0; }

// In-place-or-copy sum of count u64 words across the ranks through the host hook (one device per
// process): device -> host, hook, host -> device, synchronous on the stream.
dsi_status host_allreduce(dsi_sim *h, cudaStream_t st, const void *src, void *dst, size_t count) {
  std::vector<uint64_t> buf;
  try {
    buf.resize(count);
  } catch (...) {
    return fail(h, DSI_E_NOMEM, "host all-reduce buffer");
  }
  CUDA_TRY(h, cudaMemcpyAsync(buf.data(), src, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  if (!host_hook_sum(buf.data(), count))
    return fail(h, DSI_E_COMM, "host all-reduce hook failed");
  CUDA_TRY(h, cudaMemcpyAsync(dst, buf.data(), count * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return DSI_OK;
}

// Sum the per-config moments (and, with hist, the histograms) over every device of
// every rank: one grouped ncclAllReduce into the *_red buffers.  No-op on one device.
dsi_status sum_across(dsi_sim *h, bool hist) {
  if (!h->use_nccl) return DSI_OK;
  const size_t n_cfg = h->n_cfg;
  if (h->host_coll) {
    DeviceState &d = h->dev[0];
    dsi_status st = host_allreduce(h, d.stream, d.d_acc, d.d_red, n_cfg * dsi::NF);
    if (st == DSI_OK && hist) st = host_allreduce(h, d.stream, d.d_seg, d.d_seg_red, n_cfg * 64);
    if (st == DSI_OK && hist) st = host_allreduce(h, d.stream, d.d_si, d.d_si_red, h->si_bins_total);
    return st;
  }
  NcclApi &api = nccl();
  ncclResult_t r = api.GroupStart();
  for (auto &d : h->dev) {
    if (r != ncclSuccess) break;
    cudaSetDevice(d.ordinal);
    r = api.AllReduce(d.d_acc, d.d_red, n_cfg * dsi::NF, ncclUint64, ncclSum, d.comm, d.stream);
    if (r == ncclSuccess && hist) {
      r = api.AllReduce(d.d_seg, d.d_seg_red, n_cfg * 64, ncclUint64, ncclSum, d.comm, d.stream);
      if (r == ncclSuccess)
        r = api.AllReduce(d.d_si, d.d_si_red, h->si_bins_total, ncclUint64, ncclSum, d.comm, d.stream);
    }
  }
  const ncclResult_t r2 = api.GroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(h, DSI_E_COMM, std::string("ncclAllReduce: ") + api.GetErrorString(r != ncclSuccess ? r : r2));
  return DSI_OK;
}

namespace {
Knobs g_knobs;
}  // namespace
const Knobs &knobs() { return g_knobs; }

}  // namespace dsih

extern "C" {

dsi_status dsi_nccl_unique_id(uint8_t id[128]) {
  if (!id) return DSI_E_NULL;
  NcclApi &api = nccl();
  if (!api.ok) return DSI_E_COMM;
  ncclUniqueId u;
  if (api.GetUniqueId(&u) != ncclSuccess) return DSI_E_COMM;
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return DSI_OK;
}

dsi_status dsi_sim_comm_info(dsi_sim *h, int32_t *nranks, int32_t *rank, int32_t *transport, int32_t *cell_local) {
  if (!h || !nranks || !rank || !transport) return DSI_E_NULL;
  if (cell_local) *cell_local = cells_aligned(h) ? 1 : 0;
  *nranks = 1;
  *rank = 0;
  *transport = 0;
  if (!h->use_nccl) return DSI_OK;
  if (h->host_coll) {
    *nranks = h->opt.world;
    *rank = h->opt.rank;
    *transport = 2;
    return DSI_OK;
  }
  NcclApi &api = nccl();
  const DeviceState &d = h->dev[0];
  if (!api.CommCount || !api.CommUserRank || !d.comm) return fail(h, DSI_E_COMM, "no NCCL communicator to query");
  int n = 0, r = 0;
  if (api.CommCount(d.comm, &n) != ncclSuccess || api.CommUserRank(d.comm, &r) != ncclSuccess)
    return fail(h, DSI_E_COMM, "ncclCommCount / ncclCommUserRank failed");
  *nranks = n;
  *rank = r;
  *transport = 1;
  return DSI_OK;
}

#ifdef DSI_TEST_HOOKS
dsi_status dsi_set_host_allreduce(dsi_host_allreduce_fn fn, void *user) {
  g_host_ar = fn;
  g_host_ar_user = user;
  return DSI_OK;
}

dsi_status dsi_test_set_knob(const char *name, int32_t value) {
  if (!name) return DSI_E_NULL;
  const std::string n(name);
  if (n == "k1_fast") g_knobs.k1_fast = value;
  else if (n == "crn_two_pass") g_knobs.crn_two_pass = value;
  else if (n == "crn_threads") g_knobs.crn_threads = value;
  else if (n == "crn_sums_split") g_knobs.crn_sums_split = value;
  else if (n == "tile_r") g_knobs.tile_r = value;
  else return DSI_E_RANGE;
  return DSI_OK;
}
#endif

}  // extern "C"
