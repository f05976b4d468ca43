// Launchers for the on-device cooperative rendezvous (exchange.cu).
#pragma once

#include "cb_internal.h"

namespace cb {

constexpr int kMaxParts = 16;

// Per-part device pointers passed by value as kernel parameters.
struct PartPtrs {
  const uint32_t* src[kMaxParts];              // sender's sorted src list
  const unsigned long long* count[kMaxParts];  // its length (device)
  uint32_t* clear_bits[kMaxParts];             // sender's sampling bitmap
  uint32_t* clear_summ[kMaxParts];
  uint32_t* xbits[kMaxParts];                  // owner's exchange bitmap
  uint32_t* xsumm[kMaxParts];
  uint32_t* xprefix[kMaxParts];                // owner's exchange word ranks
  uint32_t* loc_part[kMaxParts];
  uint32_t* loc_row[kMaxParts];
};

void launch_route(const PartPtrs& pp, const uint32_t* owner, uint32_t P,
                  unsigned long long* send_counts, uint64_t max_src, cudaStream_t st);
void launch_locate(const PartPtrs& pp, const uint32_t* owner, uint32_t P, uint64_t max_src,
                   cudaStream_t st);

}  // namespace cb
