// Internal interface between fbsp.cu (single-GPU compile_batch) and shard.cu
// (the sharded compile of SURVEY §8e): the batch key format and the host-side
// helpers both need.
#pragma once
#include <vector>

#include "common.cuh"
#include "engine.h"

namespace f4b {

struct BatchFormat {
  long long D = 0;              // batch degree bound (rank space C(n + D, n))
  KeyFmt f;                     // device key format of the batch
  int KW = 1;                   // key words
  bool rank_ok = false;         // grevlex rank-bitmap path eligible (KW <= 2)
  std::vector<int32_t> cand;    // closure candidates (nonzero basis polys)
};

// Validates the rows (symbolic.py:204-225 preconditions) and picks the format.
BatchFormat batch_format(Ctx* c, long long r0, const int32_t* rb, const uint16_t* shift, const int32_t* cands,
                         long long n_cands);
// Device keys of every basis term in format f (incremental).
void encode_basis_kw(Ctx* c, const KeyFmt& f, int KW);
// Candidates in (key(LM), index) order (symbolic.py:228-235).
std::vector<int32_t> reducer_preference(Ctx* c, const std::vector<int32_t>& cand);
bool rank_path_ok_pub(const Ctx* c, int order, int n, long long D);


}  // namespace f4b
