// A16: admitted speculative actions -> scheduler job columns, on the device.
//
// Reference: Scheduler._admit_action (scheduling.py:464-511) applied, in
// batch order, to the admitted actions of many sessions entering a fresh
// scheduler, and the terms Job.utility reads (scheduling.py:59-60):
//
//   mean = EstimateBook.duration(tool)                  (scheduling.py:218-219)
//   WARM_ONLY: key (tool, "warm"), d = max(wf * mean, 1e-9), T = wf * mean
//   otherwise: key (tool, canonical_arg_hash(args)), d = max(mean, 1e-9),
//              T = mean (FULL) or wf * mean (DRY_RUN)
//   a key already held by an earlier job of the batch coalesces (no id);
//   every other action takes the next id, and is dropped when its cost
//   exceeds r_total (the id stays consumed; the dropped job holds no key, so
//   later actions of that key take ids too).
//
// Device plan:
//   * paste_live_actions flattens a live step's K-slot records (n_act per
//     session, slot-major or session-major) into action columns in batch
//     order (session, then action order) through a scan of n_act;
//   * paste_action_jobs finds each key's first action with an open-addressed
//     hash table in global memory (atomicCAS claims a slot, atomicMin keeps
//     the earliest action of an equal key), then one scan over packed
//     (first, kept) pairs gives both the id rank and the output position.
// The job columns feed paste_select_greedy (K6) directly.
#include <cub/cub.cuh>

#include "common.cuh"

namespace paste {

constexpr int JOB_T = 256;

__device__ __forceinline__ uint64_t job_key_hash(int32_t tool, bool warm, const uint8_t* key) {
  uint64_t h = 0x9e3779b97f4a7c15ull * (uint64_t)(uint32_t)(tool + 1);
  if (!warm) {
    uint64_t w0, w1;
    memcpy(&w0, key, 8);
    memcpy(&w1, key + 8, 8);
    h ^= w0 + 0x632be59bd9b4e019ull * w1;
  } else {
    h ^= 0xd6e8feb86659fd93ull;
  }
  h ^= h >> 31;
  h *= 0xbf58476d1ce4e5b9ull;
  h ^= h >> 29;
  return h;
}

__device__ __forceinline__ bool job_key_eq(const paste_actions_desc& A, int64_t i, int64_t j) {
  if (A.tool[i] != A.tool[j]) return false;
  const bool wi = A.level[i] == 1, wj = A.level[j] == 1;
  if (wi || wj) return wi == wj;
  const uint4* a = reinterpret_cast<const uint4*>(A.key + 16 * i);
  const uint4* b = reinterpret_cast<const uint4*>(A.key + 16 * j);
  const uint4 x = *a, y = *b;
  return x.x == y.x && x.y == y.y && x.z == y.z && x.w == y.w;
}

// claim / join the key's table slot; table[s] = earliest action of the key
__global__ void job_insert_kernel(paste_actions_desc A, int32_t* table, uint64_t mask,
                                  int32_t* slot_of, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_actions) return;
  const int32_t tool = A.tool[i];
  const int lv = A.level[i];
  if (tool < 0 || tool >= A.n_tools || lv < 1 || lv > 3) {
    atomicOr(bad, 1);
    slot_of[i] = -1;
    return;
  }
  uint64_t s = job_key_hash(tool, lv == 1, A.key + 16 * i) & mask;
  for (;;) {
    const int32_t cur = atomicCAS(&table[s], -1, (int32_t)i);
    if (cur == -1) break;  // new key: this action holds the slot
    if (job_key_eq(A, i, cur)) {
      atomicMin(&table[s], (int32_t)i);
      break;
    }
    s = (s + 1) & mask;
  }
  slot_of[i] = (int32_t)s;
}

// packed scan input: (takes an id) << 32 | (becomes a job)
__global__ void job_flag_kernel(paste_actions_desc A, const int32_t* table, const int32_t* slot_of,
                                int64_t* packed) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_actions) return;
  const int32_t s = slot_of[i];
  const bool first = s >= 0 && table[s] == (int32_t)i;
  // a job over r_total never enters pending_spec, so it holds no key: every
  // action of such a tool takes an id and is dropped
  const bool over = s >= 0 && (int64_t)A.cost[A.tool[i]] > A.r_total;
  packed[i] = ((int64_t)(first || over) << 32) | (int64_t)(first && !over);
}

__device__ __forceinline__ double py_max_clamp(double x) {  // Python max(x, 1e-9)
  return 1e-9 > x ? 1e-9 : x;
}

__global__ void job_write_kernel(paste_actions_desc A, const int64_t* packed_in,
                                 const int64_t* excl, paste_jobs_out J) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = A.n_actions;
  if (i > n) return;
  if (i == n) {  // totals
    const int64_t last = n ? excl[n - 1] + packed_in[n - 1] : 0;
    *J.n_jobs = last & 0xffffffffll;
    *J.next_id = A.id_base + (last >> 32);
    return;
  }
  const int64_t v = packed_in[i];
  if (!(v & 1)) return;
  const int64_t pos = excl[i] & 0xffffffffll, rank = excl[i] >> 32;
  const int32_t tool = A.tool[i];
  const int lv = A.level[i];
  const double mean = A.mean[tool], wf = A.warm_fraction;
  const double warm = __dmul_rn(wf, mean);
  double dur, bene;
  if (lv == 1) {
    dur = py_max_clamp(warm);
    bene = warm;
  } else {
    dur = py_max_clamp(mean);
    bene = lv == 3 ? mean : warm;
  }
  J.p[pos] = A.p[i];
  J.benefit[pos] = bene;
  J.duration[pos] = dur;
  J.cost[pos] = A.cost[tool];
  J.id[pos] = A.id_base + rank;
  if (J.action) J.action[pos] = i;
}

// live records -> flattened action columns (batch order)
__global__ void live_count_kernel(int64_t n, const int32_t* n_act, int64_t* cnt) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) cnt[s] = n_act[s];
}

__global__ void live_flatten_kernel(paste_live_actions_desc L, const int64_t* cnt,
                                    const int64_t* excl) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = L.n_sessions;
  if (s > n) return;
  if (s == n) {
    *L.n_actions = n ? excl[n - 1] + cnt[n - 1] : 0;
    return;
  }
  const paste_predict_out& o = L.out;
  const int na = (int)cnt[s];
  const int64_t base = excl[s];
  for (int a = 0; a < na; ++a) {
    const int64_t slot = out_at(o, n, s, a);
    const int pr = o.act_pred[slot];
    const int64_t pslot = out_at(o, n, s, pr);
    const int pat = o.pred_pat[pslot];
    const paste_pattern P = L.pool.patterns[pat];
    const int64_t j = base + a;
    L.tool[j] = P.target_tool;
    L.level[j] = o.act_level[slot];
    L.p[j] = P.p;
    L.session[j] = s;
    L.slot[j] = (int32_t)slot;
    if (L.key) {
      const uint4* src = reinterpret_cast<const uint4*>(L.slot_keys + 16 * slot);
      reinterpret_cast<uint4*>(L.key)[j] = *src;
    }
  }
}

}  // namespace paste

using namespace paste;

static int64_t table_size(int64_t n) {
  int64_t t = 1024;
  while (t < 2 * n) t <<= 1;
  return t;
}

extern "C" int64_t paste_action_jobs_scratch_bytes(int64_t n_actions) {
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_actions > 0 ? n_actions : 1));
  return 4 * table_size(n_actions) + 4 * n_actions + 16 * n_actions + (int64_t)cub_bytes + 1024;
}

extern "C" int paste_action_jobs(const paste_actions_desc* a, paste_jobs_out* j, void* scratch,
                                 int64_t scratch_bytes, void* stream_) {
  reset_launches();
  PASTE_REQUIRE(a != nullptr && j != nullptr, "null descriptor");
  PASTE_REQUIRE(j->n_jobs && j->next_id, "n_jobs / next_id outputs required");
  const int64_t n = a->n_actions;
  PASTE_REQUIRE(n >= 0 && n < (1ll << 31), "n_actions out of range");
  PASTE_REQUIRE(n == 0 || (a->tool && a->level && a->p && a->key && a->mean && a->cost),
                "null action column");
  const int64_t need = paste_action_jobs_scratch_bytes(n);
  PASTE_REQUIRE(scratch != nullptr && scratch_bytes >= need, "scratch too small (%lld bytes)",
                (long long)need);
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t T = table_size(n);
  uint8_t* s = static_cast<uint8_t*>(scratch);
  int32_t* table = reinterpret_cast<int32_t*>(s);
  s += 4 * T;
  int* bad = reinterpret_cast<int*>(s);
  s += 256;
  int32_t* slot_of = reinterpret_cast<int32_t*>(s);
  s += (4 * n + 255) / 256 * 256;
  int64_t* packed = reinterpret_cast<int64_t*>(s);
  s += 8 * n;
  int64_t* excl = reinterpret_cast<int64_t*>(s);
  s += 8 * n;
  void* cub_tmp = s;
  size_t cub_bytes = (size_t)(static_cast<uint8_t*>(scratch) + scratch_bytes - s);
  PASTE_CUDA_CHECK(cudaMemsetAsync(table, 0xff, 4 * T, stream));
  PASTE_CUDA_CHECK(cudaMemsetAsync(bad, 0, 4, stream));
  const int blocks = (int)((n + JOB_T) / JOB_T);  // n + 1 threads for the totals
  if (n > 0) {
    job_insert_kernel<<<blocks, JOB_T, 0, stream>>>(*a, table, (uint64_t)(T - 1), slot_of, bad);
    job_flag_kernel<<<blocks, JOB_T, 0, stream>>>(*a, table, slot_of, packed);
    PASTE_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, packed, excl, (int)n, stream));
    count_launch(3);
  }
  job_write_kernel<<<blocks, JOB_T, 0, stream>>>(*a, packed, excl, *j);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  int h_bad = 0;
  PASTE_CUDA_CHECK(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, stream));
  PASTE_CUDA_CHECK(cudaStreamSynchronize(stream));
  if (h_bad) {
    set_error("action tool id outside the tool table or level outside 1..3");
    return PASTE_ERR_INVALID;
  }
  return PASTE_OK;
}

extern "C" int64_t paste_live_actions_scratch_bytes(int64_t n_sessions) {
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_sessions > 0 ? n_sessions : 1));
  return 16 * n_sessions + (int64_t)cub_bytes + 512;
}

extern "C" int paste_live_actions(const paste_live_actions_desc* l, void* scratch,
                                  int64_t scratch_bytes, void* stream_) {
  reset_launches();
  PASTE_REQUIRE(l != nullptr && l->n_actions != nullptr, "null descriptor");
  const int64_t n = l->n_sessions;
  PASTE_REQUIRE(n >= 0 && n < (1ll << 31), "n_sessions out of range");
  const int64_t need = paste_live_actions_scratch_bytes(n);
  PASTE_REQUIRE(scratch != nullptr && scratch_bytes >= need, "scratch too small (%lld bytes)",
                (long long)need);
  cudaStream_t stream = (cudaStream_t)stream_;
  uint8_t* s = static_cast<uint8_t*>(scratch);
  int64_t* cnt = reinterpret_cast<int64_t*>(s);
  s += 8 * n;
  int64_t* excl = reinterpret_cast<int64_t*>(s);
  s += 8 * n;
  size_t cub_bytes = (size_t)(static_cast<uint8_t*>(scratch) + scratch_bytes - s);
  const int blocks = (int)((n + JOB_T) / JOB_T);
  if (n > 0) {
    live_count_kernel<<<blocks, JOB_T, 0, stream>>>(n, l->out.n_act, cnt);
    PASTE_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(s, cub_bytes, cnt, excl, (int)n, stream));
    count_launch(2);
  }
  live_flatten_kernel<<<blocks, JOB_T, 0, stream>>>(*l, cnt, excl);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
