// glu_internal.h -- layouts shared by the host plan builder and the device
// kernels.  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <string>

struct glu_plan;

namespace glu {

enum ItemKind : int32_t {
    kPush = 0,  // destination segment, ordered chunks, lanes over chunk entries
    kDeep = 1,  // one target slot with many ordered contributions (hub rows)
};

// One warp task in one phase.  32 bytes so a warp fetches it with two
// 16-byte loads.
struct alignas(16) Item {
    int64_t map_off;  // kPush: first uint16 map entry; kDeep: first DeepRef
    int32_t base;     // kPush: absolute slot of the segment start; kDeep: target slot
    int32_t span;     // kPush: positions covered by the segment (<= 65535); kDeep: 1
    int32_t c0, c1;   // kPush: chunk range
    int32_t macs;     // MACs carried
    int32_t kind;     // ItemKind
};
static_assert(sizeof(Item) == 32, "Item layout");

// A contiguous run of one source column's L entries, applied with one
// multiplier.  16 bytes: one vector load.  meta = cnt | kEpochBit when the
// chunk shares a target with an earlier chunk of the same epoch of its item,
// i.e. the warp must finish every earlier chunk's stores before this one.
constexpr int32_t kEpochBit = int32_t(0x80000000u);
struct alignas(16) Chunk {
    int32_t m;     // slot of U(j,k): the multiplier
    int32_t d;     // slot of A_s(j,j): the pivot
    int32_t p0;    // first L slot of the run
    int32_t meta;  // entries in the run | kEpochBit
};
static_assert(sizeof(Chunk) == 16, "Chunk layout");

// One contribution of a kDeep item: target -= (v[l] / v[d]) * v[m].
struct alignas(16) DeepRef {
    int32_t l, d, m, pad;
};
static_assert(sizeof(DeepRef) == 16, "DeepRef layout");

struct glu_plan_view {
    int64_t n_levels;
    const int64_t *level_item_ptr;
    const Item *items;
    int64_t n_items;
    const Chunk *chunks;
    int64_t n_chunks;
    int64_t n_map;
    const DeepRef *deep;
    int64_t n_deep;
};

const glu_plan_view plan_view(const glu_plan *p);
void set_error(const std::string &s);

}  // namespace glu
