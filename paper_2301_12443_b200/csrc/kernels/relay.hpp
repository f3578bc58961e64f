// Internal interface of the K11 peer relay kernels (relay.cu).
#pragma once

#include <cuda_runtime.h>

namespace pbdk {

constexpr int kRelayMaxPeers = 16;

// spin until flags[i] >= *seq + bias for i < count
struct RelayWaitArgs {
  const unsigned long long* flags[kRelayMaxPeers];
  const unsigned long long* seq;
  unsigned long long bias;
  int count;
};

// dst[m][0:16*vec16[m]) = src[m][...]; then ready[m] = *seq + 1 and *seq += 1
struct RelayCopyArgs {
  const void* src[kRelayMaxPeers];
  void* dst[kRelayMaxPeers];
  long long vec16[kRelayMaxPeers];
  unsigned long long* ready[kRelayMaxPeers];
  unsigned long long* seq;
  unsigned int* ticket;
  int count;
};

// advance: *seq += 1; then flags[i] = *seq (peer stores, system scope)
struct RelayReleaseArgs {
  unsigned long long* flags[kRelayMaxPeers];
  unsigned long long* seq;
  int count;
  int advance = 1;
};

int relay_wait(const RelayWaitArgs& a, cudaStream_t st);
int relay_copy(const RelayCopyArgs& a, int ctas, cudaStream_t st);
int relay_release(const RelayReleaseArgs& a, cudaStream_t st);

// ---- DP-group gradient sharing over peer memory (fused with the SGD update, bd_kernels.cu)
constexpr int kDpMaxGroup = 8;

}  // namespace pbdk
