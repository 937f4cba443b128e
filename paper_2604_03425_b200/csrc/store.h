// store.h -- wire / disk format of bundles and keys with streaming transfer (store.cu).
#pragma once

#include <string>

#include "common.cuh"

namespace aegis {

class Context;
struct Bundle;

void store_save_bundle(Context& c, const Bundle& b, const std::string& path);
Bundle* store_load_bundle(Context& c, const std::string& path);
void store_save_key(Context& c, u64 key_id, const std::string& path);
void store_load_key(Context& c, u64 key_id, const std::string& path);

}  // namespace aegis
