// Device empty-grating setup (empty.cu): per-context state release.
#pragma once
#include "ctx.cuh"

namespace ps {
void empty_release(Ctx* c);
}  // namespace ps
