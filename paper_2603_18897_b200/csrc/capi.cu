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
