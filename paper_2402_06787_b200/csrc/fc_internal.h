// Internal layout shared by the host API (fc_api.cu) and the kernel
// (fc_kernel.cu).  Not part of the C ABI.
#pragma once
#include <stdint.h>

#include "../../include/forestcoll.h"

#define FC_MAXR FC_MAX_RANKS
#define FC_ALIGN 128          // chunk boundaries / scratch phase alignment (bytes)
#define FC_READY_WORDS 64     // 64-bit ready slot per peer r at words [2r, 2r+1]:
                              // entry epoch (low) | output-buffer tag (high)
#define FC_TABLE_MAGIC 0x50434c46  // 'FLCP'
#define FC_TABLE_VERSION 1
#define FC_HEADER_WORDS 16
#define FC_RANKDESC_WORDS 8
#define FC_TASK_WORDS 128

// Task kinds (one task = one tree as seen from one rank).  See DESIGN.md §3.
enum {
  FC_K_AG_ROOT = 1,  // allgather root: send -> own recv + AG children
  FC_K_AG_FWD = 2,   // allgather interior: wait parent, recv -> AG children
  FC_K_RS_FWD = 3,   // reduce-scatter non-root: own + children partials -> parent scratch
  FC_K_RS_ROOT = 4,  // reduce-scatter root: own + children partials -> out
  FC_K_AR_ROOT = 5,  // allreduce root: reduce, write own buf, push to AG children
  FC_K_WAIT_AG = 6,  // allgather leaf: wait for the chunk (completion only)
};

// Task word offsets.
enum {
  TW_KIND = 0,
  TW_TREE = 1,
  TW_STAGE = 2,
  TW_ROOT = 3,
  TW_MLO = 4,
  TW_MHI = 5,
  TW_AG_PARENT = 6,
  TW_N_AG_CHILD = 7,
  TW_AG_CHILD = 8,     // [FC_MAXR]
  TW_RS_PARENT = 24,
  TW_RS_PSLOT = 25,
  TW_RS_PPREFIX = 26,
  TW_N_RS_CHILD = 27,
  TW_RS_CHILD = 28,    // [FC_MAXR]
  TW_RS_CSLOT = 44,    // [FC_MAXR]
  TW_RS_CPREFIX = 60,  // [FC_MAXR]
  TW_LAG = 76,         // dense stage index: claim-order skew (chunk + lag * TW_LAG)
  TW_AG_LEAFMASK = 77, // bit j: AG child j is a leaf (gets an arrival count, no chunk flags)
  TW_AG_MYSLOT = 78,   // LL protocol: staging slot receiving this tree here (-1 at the root)
  TW_AG_MYPREFIX = 79,
  TW_AG_CSLOT = 80,    // [FC_MAXR] children's staging slots
  TW_AG_CPREFIX = 96,  // [FC_MAXR]
  TW_END = 112,
};

// Header word offsets of a plan table (see compiler.py for the writer).
enum {
  TH_MAGIC = 0,
  TH_VERSION = 1,
  TH_COLLECTIVE = 2,
  TH_NRANKS = 3,
  TH_K = 4,
  TH_NTREES = 5,
  TH_NTASKS = 6,
  TH_TASK_WORDS = 7,
  TH_MAX_SLOT_UNITS = 8,
  TH_MAX_SLOTS = 9,
  TH_MAX_AG_SLOT_UNITS = 10,
  TH_MAX_AG_SLOTS = 11,
  TH_FLAGS = 12,
};
// TH_FLAGS bits (compiler.py computes them from the schedule alone).
// FC_PLAN_ONEHOP: every logical edge of the forest is one path through the
// same switch [src, sw, dst], and every rank sends exactly (N-1)*k units.
// Then each GPU has an uplink and a downlink to that switch, and a depth-1
// all-to-all uses every link exactly as much as the forest does (same T*):
// the one-hop allgather and the one-shot reductions may replace the forest.
#define FC_PLAN_ONEHOP 1
// Rank descriptor words: first task, n active, n wait, slot units, n slots.
enum { RD_FIRST = 0, RD_NACTIVE = 1, RD_NWAIT = 2, RD_SLOT_UNITS = 3, RD_NSLOTS = 4 };

// Per-rank control block at the head of each rank's workspace.
struct FcCtl {
  unsigned int epoch;  // number of completed launches
  unsigned int claim;  // dynamic work-claim counter (reset by the last CTA)
  unsigned int done;   // CTAs finished in the current launch
  unsigned int error;  // sticky device error code (0 = ok)
  unsigned int info[12];
};

#define FC_DEVERR_TIMEOUT_AG 1
#define FC_DEVERR_TIMEOUT_RS 2
#define FC_DEVERR_TIMEOUT_READY 3
#define FC_DEVERR_BUFFER_MISMATCH 4  // peers passed differently registered outputs

// One record per executed item when tracing is enabled (fc_comm_set_trace).
struct FcTraceRec {
  unsigned long long t_start, t_end;  // %globaltimer ns: claim .. published
  unsigned t_wait;                    // ns spent waiting on flags / readiness
  unsigned t_move;                    // ns from ready to data moved (before publish)
  int chunk;
  short rank, task;
  short worker;
  unsigned short launch;  // epoch (low 16 bits)
  unsigned peer_bytes;    // bytes this item stored into other ranks' memory
                          // (payload + LL128 line tags + flag words)
};

struct FcParams {
  int nranks;
  int nlocal;
  int ctas_per_rank;
  int k;
  int local_rank[FC_MAXR];
  const int* tasks[FC_MAXR];  // by local index: this rank's task rows
  int nactive[FC_MAXR];
  int nwait[FC_MAXR];
  int lag_max[FC_MAXR];       // by local index: max TW_LAG over active tasks
  FcCtl* ctl[FC_MAXR];        // by local index
  // by rank: this process's view (peer-mapped for remote ranks)
  const char* send[FC_MAXR];  // only local ranks are dereferenced
  char* recv[FC_MAXR];        // AG/AR: peer-mapped; RS: local only
  char* scratch[FC_MAXR];
  unsigned int* flags[FC_MAXR];
  long long shard_elems;   // S: elements per root shard
  long long stride_elems;  // distance between root shards in the N-shard buffer
  long long total_elems;   // elements in the N-shard buffer (AR: count)
  long long unit_bytes;    // scratch bytes per unit of tree multiplicity per window
  long long timeout_ns;
  int esize;
  int dtype;
  int op;       // FC_SUM or FC_AVG
  float scale;  // FC_AVG: fp32 1/N applied once by tree roots
  unsigned long long tag;  // identity of the peer-mapped output (registration, offset, size)
  int nchunks;  // chunks per tree slice for the whole call
  int tail;     // chunk-flag protocol: the last `tail` chunks halve in size, step by step
  int c0, c1;   // chunk window of this launch
  int maxc;     // flag stride per tree / slot
  int cnt_off;      // word offset of per-tree leaf arrival counters
  int ag_flag_off;  // word offset of AG flags in the flags region
  int rs_flag_off;  // word offset of RS flags in the flags region
  int lag;          // claim-order skew in chunks per stage
  int copy_mode;    // 0: TMA bulk stores, 1: bulk loads + 16-byte lane stores
  int root_local_done;  // allgather: own shard already placed in recv (DMA engine)
  int worker_warps;     // warps per worker (1, 2, 4, 8): items in flight per CTA = 8 / this
  int proto;            // 0: chunk flags + fences, 1: LL128 lines (flag in every 128 B)
  int pdl;              // launch with programmatic stream serialization
  long long ll_unit_bytes;  // LL: staging bytes per unit multiplicity per window
  long long ll_ag_base;     // LL: offset of the broadcast staging within the LL region
  long long ll_region_off;  // LL: offset of the (zeroed, dedicated) LL region from scratch
  long long ll_half;        // LL: the region's two halves alternate by launch-epoch parity
  FcTraceRec* trace;
  unsigned* trace_count;
  unsigned trace_cap;
};

// NVLS (NVSwitch multicast) engine: executes a ForestColl forest whose
// NVSwitch hops are pruned for multicast / in-switch aggregation
// (schedule.py:237-306): every root writes its shard once into the switch.
struct FcNvlsParams {
  int nranks, rank, mode, dtype;  // mode: 0 allgather, 1 reduce-scatter, 2 allreduce
  int op;                         // FC_SUM or FC_AVG
  float scale;                    // FC_AVG: fp32 1/N
  int bar_off;                    // word offset of the NVLS barrier words (2 * FC_MAXR)
  FcCtl* ctl;
  unsigned int* flags[FC_MAXR];
  char* mc;                       // multicast VA of the pool (+ buffer offset)
  const char* send;               // allgather source (any device buffer)
  char* out;                      // reduce-scatter destination (any device buffer)
  long long shard_bytes;          // bytes per root shard
  long long total_bytes;          // bytes of the N-shard buffer in the pool
  long long timeout_ns;
  // mode 3 (allgather, LL over multicast): staging at the top of the pool,
  // two halves alternating by epoch parity; 16-byte units {d0, e, d1, e}
  char* mc_stage;                 // multicast VA of the staging region
  const char* uc_stage;           // this GPU's view of the same region
  long long ll_half;              // bytes per half
  // modes 4 (reduce-scatter) / 5 (allreduce), LL over multicast + one-shot
  const int* os_trees;            // [os_ntrees][FC_OS_TREE_WORDS]
  int os_ntrees, k;
  long long buf_bytes;            // bytes of each rank's input buffer
  long long count;                // AR: elements of the buffer
  long long shard_elems;          // elements per root shard
  // one-shot without multicast (tree-engine communicators, modes 6/7/8): LL128
  // lines go to every rank's staging through its peer mapping.  One grid
  // serves `nlocal` ranks (several in virtual mode, cooperative launch):
  // CTAs [i*ctas_per_rank, (i+1)*ctas_per_rank) run local rank lrank[i].
  char* peer_stage[FC_MAXR];
  int nlocal, ctas_per_rank;
  int lrank[FC_MAXR];
  FcCtl* lctl[FC_MAXR];
  const char* lsend[FC_MAXR];
  char* lout[FC_MAXR];
};

// One tree of a reduce-scatter / allreduce forest for the NVLS engine's
// one-shot LL reduction: every rank holds every rank's input after one
// multicast hop and evaluates the in-tree locally in the executor's order
// (post-order; own value + children ascending; one rounding per node).
#define FC_OS_TREE_WORDS (4 + FC_MAXR + FC_MAXR + FC_MAXR * FC_MAXR)
enum { OS_ROOT = 0, OS_MLO = 1, OS_MHI = 2, OS_NPOST = 3, OS_POST = 4,
       OS_NCH = 4 + FC_MAXR, OS_CH = 4 + 2 * FC_MAXR };

// Kernel entry (fc_kernel.cu).  Returns a cudaError_t value.
int fc_launch(const FcParams& p, int reduce_dtype, int cooperative,
              void* stream, int* grid_out);
int fc_max_ctas_per_sm(int reduce_dtype, int* out);
int fc_warps_per_cta();
int fc_nvls_launch(const FcNvlsParams& p, int ctas, void* stream);
// grid size for the one-shot kernels (modes 6/7/8): every CTA co-resident
int fc_oneshot_max_ctas(int mode, int dtype, int nranks, int* out);

// Copy-engine path of the 2-rank forest (fc_ce.cu).  Its flag slots are
// 64-bit words at the end of each rank's flag area: FC_CE_READY + r holds
// rank r's entry (tag << 32 | epoch), FC_CE_DONE + r its exit epoch.
#define FC_CE_READY 0
#define FC_CE_DONE FC_MAXR
#define FC_CE_SLOTS (2 * FC_MAXR)
struct FcCeParams {
  FcCtl* ctl;                      // own control block (epoch, sticky error)
  unsigned long long* my_slots;    // own CE slots
  unsigned long long* peer_slots;  // the peer's CE slots (mapped)
  unsigned long long tag;          // identity of the output buffer (as FcParams.tag)
  long long timeout_ns;
  int me, peer;
  int phase;                       // 0: entry handshake, 1: exit handshake
};
int fc_ce_sync_launch(const FcCeParams& p, void* stream);
int fc_ce_copy_launch(void* dst, const void* src, long long n, int ctas, void* stream);
