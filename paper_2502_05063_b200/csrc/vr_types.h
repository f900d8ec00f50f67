// vr_types.h — plain data types shared by the device code (vr_common.cuh) and the host-side
// interfaces (vr_internal.h).
#pragma once
#include <cstdint>

namespace vr {

// The clearing set of a dimension in the output-sensitive mode: the cidx of its columns that
// are pivots (deaths) of the dimension below, in an open-addressing table of 64-bit keys
// (~0 = empty slot, linear probing), fronted by a blocked Bloom filter — one 32-bit word per
// key with 3 bits set — that answers most of the (mostly negative) membership probes from a
// few MB that stay in L2 (vr_common.cuh set_put / set_has).
struct ClearSet {
  uint64_t* table;       // nullptr: no set
  uint64_t mask;         // table slots - 1 (power of two)
  uint32_t* bloom;
  uint32_t bloom_words;  // >= 1
};

}  // namespace vr
