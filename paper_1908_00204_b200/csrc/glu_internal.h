// glu_internal.h -- layouts shared by the host plan builder and the device
// kernels.  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

struct glu_plan;

namespace glu {

enum ItemKind : int32_t {
    kPush = 0,  // destination segment, ordered chunks, lanes over chunk entries
    kDeep = 1,  // one target slot with many ordered contributions (hub rows)
};

constexpr int kMaxItemMacs = 128;   // push item: at most 4 entries per lane
constexpr int kMaxItemChunks = 32;  // push item: one chunk descriptor per lane

// One warp task in one phase.  48 bytes = three 16-byte loads.
//   kPush: the MACs of one phase into a set of <= 256 distinct targets of one
//          destination column k, given as ordered chunks; per MAC a u8 index
//          into the item's sorted target list (u16 offsets from `base`).
//          The warp stages the targets in shared memory, applies the chunks
//          in order and writes each target back once.
//   kDeep: one target with many ordered contributions (power/ground rows).
struct alignas(16) Item {
    int64_t map_off;  // kPush: first u8 map entry; kDeep: first DeepRef
    int64_t tgt_off;  // kPush: first u16 target offset
    int32_t base;     // kPush: slot the target offsets are relative to; kDeep: target slot
    int32_t c0;       // kPush: first chunk
    int32_t nch;      // kPush: chunks (<= kMaxItemChunks)
    int32_t ntgt;     // kPush: distinct targets (<= kMaxItemMacs)
    int32_t macs;     // MACs carried
    int32_t kind;     // ItemKind | critical << 1 | phase << 2
    int32_t col;      // first entry of its ColDep list (destination columns)
    int32_t need;     // number of destination columns (1..4)
};

// A destination column of an item and the number of items into that column
// in earlier phases (the item's dataflow dependency on its own targets).
struct ColDep {
    int32_t col, need;
};
static_assert(sizeof(Item) == 48, "Item layout");

// A contiguous run of one source column's L entries, applied with one
// multiplier.  16 bytes: one vector load.  meta = cnt | kEpochBit when the
// chunk shares a target with an earlier chunk of the same epoch of its item,
// i.e. the warp must finish every earlier chunk's stores before this one.
constexpr int32_t kEpochBit = int32_t(0x80000000u);
struct alignas(16) Chunk {
    int32_t m;     // slot of U(j,k): the multiplier
    int32_t d;     // while building: slot of A_s(j,j) (the pivot); in the plan: source column j
    int32_t p0;    // first L slot of the run
    int32_t meta;  // entries in the run | kEpochBit
};
static_assert(sizeof(Chunk) == 16, "Chunk layout");

// One contribution of a kDeep item: target -= (v[l] / v[d]) * v[m].
struct alignas(16) DeepRef {
    int32_t l, d, m, pad;
};
static_assert(sizeof(DeepRef) == 16, "DeepRef layout");

// ---------------------------------------------------------------------------
// Supernodal engine (glu_snode.cpp / glu_snode.cu): the plan for patterns
// whose per-MAC plan above does not fit (cfg4: 3.8e10 MACs).  Columns are
// grouped into fundamental supernodes S = [s0, s1) (L(:,c-1) = {c} u L(:,c),
// U(c-1,c) != 0), whose columns share the rows R_S below the supernode, and
// cut into panels of <= kSnW columns.  Index records are 16-byte vectors.
// ---------------------------------------------------------------------------
constexpr int kSnW = 16;  // panel width: one warp lane per panel column / row
// RG tasks stage their target slots, the pushes' L rows and their MAC
// indices in a warp's shared memory
constexpr int kRgPushes = 16;   // pushes per RG task
constexpr int kRgSlots = 512;   // distinct slots (targets and multipliers U(p0, k))
constexpr int kRgIdx = 2048;    // MAC indices (u16)
constexpr int kRgRows = 512;    // L rows (a push has at most kRgRows / 4 rows below its column)

struct alignas(16) I4 {
    int32_t x, y, z, w;
};

// task code = record.x >> 27 = kind << 2 | flags
enum SnTaskKind : int32_t {
    kSnTrsm = 0,  // rows below a panel: factor its diagonal block locally, divide, in-panel updates
    kSnRect = 1,  // push rows below the source panel into every column of the target panel
    kSnUw = 2,    // write the solved U(P, K) of a push whose RECT chunks all read it
    kSnRg = 3,    // a run of one-chunk pushes from one-column panels into one target panel
    kSnWb = 4,    // write a panel's factored diagonal block back in place
};
enum SnTaskFlags : int32_t {
    kSnTriF = 1,    // RECT: forward substitution of U(P, K) inside the source block first
    kSnWriteU = 2,  // RECT: the only reader of U(P, K) -- it writes the solved values
};

struct SnPlan {
    int64_t n = 0, nnz = 0;
    std::vector<I4> sn;      // {s0, s1, |R_S|, first pair}
    std::vector<I4> pan;     // {p0, p1, supernode, rows below the panel}
    std::vector<I4> panm;    // per panel {pushes' RECT chunks into it, TRSM chunks, scratch offset | -1,
                             //  WB + UW tasks after which its values are final}
    std::vector<I4> pairs;   // per (supernode S, target column k): {k, a, base, map}
    std::vector<int32_t> relmap;  // positions of R_S's rows in column k (absolute slots)
    std::vector<I4> push;    // {source panel, first pair, end pair, target panel}, target-major
    std::vector<int32_t> push_need;  // per push: RECT chunks of earlier pushes into its target
    // 3 records per task, in a topological (as-soon-as-possible) order:
    //   {code << 27 | chunk, source panel P, p0, p1}, {s1, rows below p1, pair0, pair1},
    //   {target panel K, need, 0, 0}; RG: {code << 27 | pushes, first MAC index, first U index, chunks},
    //   {first slot, slots, first push, pushes}, {K, need, 0, 0}
    std::vector<I4> tasks;
    std::vector<float> task_cost;    // per task: the latency model's cost (us), for the warp assignment
    std::vector<int64_t> col_ptr_h;  // the pattern's column pointers (host copy-out of final panels)
    std::vector<int32_t> col_a;      // per column c: first row of c's supernode present in c
    // RG tasks: per RG {first slot, slots, first MAC index, first U index}; the
    // slots it stages in shared memory (targets and multipliers); per MAC
    // (push, pair q, row t at q * h + t) the index of its target in that
    // list; per (push, pair) the index of U(p0, k)
    std::vector<I4> rg;
    std::vector<int32_t> rg_chunks;  // per RG: RECT chunks its pushes count for
    std::vector<int32_t> rg_slot;
    std::vector<uint16_t> rg_idx, rg_uidx;
    int64_t n_dblk = 0;              // doubles of factored-diagonal-block scratch (panels w >= 2)
    int64_t crit_ns = 0;             // critical path of the plan's latency model
    int64_t macs = 0;
};

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
    const uint8_t *map8;
    const uint16_t *tgt16;
    int64_t n_tgt;
    const int32_t *col_total;  // per column: items into it (all phases)
    int64_t tail_t0;           // columns >= tail_t0: dense cluster tail (n: none)
    const ColDep *cdeps;
    int64_t n_cdeps;
    int64_t max_push_macs;     // largest push item (selects the kernel variant)
    const SnPlan *sn;          // supernodal engine (no items above), or null
};

const glu_plan_view plan_view(const glu_plan *p);
// glu_snode.cpp: builds the supernodal plan; GLU_OK, GLU_MISMATCH or GLU_EINVAL
int64_t sn_build(int64_t n, const int64_t *col_ptr, const int64_t *row_idx, const int64_t *diag_pos,
                 const int64_t *row_ptr, const int64_t *col_idx, const int64_t *csc_pos,
                 int n_threads, SnPlan *out);
void set_error(const std::string &s);

// glu_snode.cu: device side of the supernodal engine
struct SnDev;
int64_t sn_upload(const SnPlan *p, SnDev **out, int64_t *bytes);
void sn_free(SnDev *d);
int sn_grid(int sm_count);
int64_t sn_set_trace(SnDev *d, int mode);
// Copies the values of v to the host while the factorization launched on s
// runs (the column ranges whose panels are final), the rest once s is done.
int64_t sn_copy_out(SnDev *d, const double *v, double *out, void *stream);
int64_t sn_read_trace(SnDev *d, int64_t *out, int64_t max_tasks);
// one factorization of v (A_s values after the scatter); pivot failures
// are min-reduced into *fail as (fail_level << 32 | column) or column
int64_t sn_launch(SnDev *d, double *v, const int32_t *col_ptr, const int32_t *diag_pos,
                  const int32_t *fail_level, int32_t n, double thresh, bool by_column,
                  unsigned long long *fail, int *err, void *stream);

}  // namespace glu
