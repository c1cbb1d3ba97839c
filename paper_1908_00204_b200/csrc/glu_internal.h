// glu_internal.h -- layouts shared by the host plan builder and the device
// kernels.  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <string>

struct glu_plan;

namespace glu {

// One warp task: a destination-column segment in one phase.  32 bytes so a
// warp fetches it with two 16-byte loads.
struct alignas(16) Item {
    int64_t map_off;  // first uint16 map entry of this item
    int32_t base;     // absolute slot of the segment's first position
    int32_t span;     // positions covered by the segment (<= 65535)
    int32_t c0, c1;   // chunk range
    int32_t macs;     // MACs carried (= map entries)
    int32_t pad;
};
static_assert(sizeof(Item) == 32, "Item layout");

// A contiguous run of one source column's L entries, applied with one
// multiplier.  16 bytes: one vector load.
struct alignas(16) Chunk {
    int32_t m;    // slot of U(j,k): the multiplier
    int32_t d;    // slot of A_s(j,j): the pivot
    int32_t p0;   // first L slot of the run
    int32_t cnt;  // entries in the run
};
static_assert(sizeof(Chunk) == 16, "Chunk layout");

struct glu_plan_view {
    int64_t n_levels;
    const int64_t *level_item_ptr;
    const Item *items;
    int64_t n_items;
    const Chunk *chunks;
    int64_t n_chunks;
    int64_t n_map;
};

const glu_plan_view plan_view(const glu_plan *p);
void set_error(const std::string &s);

}  // namespace glu
