// C-ABI plumbing shared by every libpaste entry point: thread-local last
// error, launch counting (reported by bench.py as gpu_launches).
#include "common.cuh"

namespace paste {

static thread_local char g_last_error[1024] = "";
static thread_local int g_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

void count_launch(int n) { g_launches += n; }
void reset_launches() { g_launches = 0; }

}  // namespace paste

extern "C" const char* paste_last_error(void) { return paste::g_last_error; }
extern "C" int paste_abi_version(void) { return PASTE_ABI_VERSION; }
extern "C" int paste_last_launch_count(void) { return paste::g_launches; }

// A batch of async copies on one stream in one call (the serving loop's
// sized record downloads and input uploads: one ctypes call per step side).
extern "C" int paste_memcpy_batch(int32_t n, void* const* dst, const void* const* src,
                                  const int64_t* bytes, int32_t kind, void* stream) {
  using namespace paste;
  PASTE_REQUIRE(n >= 0 && (n == 0 || (dst && src && bytes)), "null copy list");
  PASTE_REQUIRE(kind == PASTE_COPY_H2D || kind == PASTE_COPY_D2H || kind == PASTE_COPY_D2D,
                "unknown copy kind");
  const cudaMemcpyKind k = kind == PASTE_COPY_H2D   ? cudaMemcpyHostToDevice
                           : kind == PASTE_COPY_D2H ? cudaMemcpyDeviceToHost
                                                    : cudaMemcpyDeviceToDevice;
  for (int32_t i = 0; i < n; ++i)
    if (bytes[i] > 0)
      PASTE_CUDA_CHECK(cudaMemcpyAsync(dst[i], src[i], (size_t)bytes[i], k, (cudaStream_t)stream));
  return PASTE_OK;
}
