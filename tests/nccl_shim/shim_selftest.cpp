// CPU self-test of the NCCL test shim (built with -DSHIM_HOST_TEST, run by
// tests/test_nccl_shim.py): N forked ranks run in-place all-reduce sum / max and a grouped
// pairwise exchange larger than one mailbox (chunk interleaving), checking every value.
#include <nccl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <sys/wait.h>
#include <unistd.h>

#include <vector>

static int run_rank(ncclUniqueId id, int N, int r) {
  ncclComm_t c;
  if (ncclCommInitRank(&c, N, id, r) != ncclSuccess) return 1;
  int bad = 0;
  const size_t M = 300000;  // > 1 MiB mailbox in doubles -> several chunks
  for (int rep = 0; rep < 3; ++rep) {
    std::vector<double> v(M);
    for (size_t i = 0; i < M; ++i) v[i] = (i % N == (size_t)r) ? (double)(i + rep) : 0.0;
    ncclAllReduce(v.data(), v.data(), M, ncclFloat64, ncclSum, c, nullptr);
    for (size_t i = 0; i < M; ++i) bad += v[i] != (double)(i + rep);
    std::vector<uint64_t> u(1000);
    for (size_t i = 0; i < u.size(); ++i) u[i] = i * N + r;
    ncclAllReduce(u.data(), u.data(), u.size(), ncclUint64, ncclMax, c, nullptr);
    for (size_t i = 0; i < u.size(); ++i) bad += u[i] != i * N + N - 1;
    // pairwise exchange with partner r ^ 1 (as libtanq's remap: GroupStart, Send, Recv, GroupEnd)
    const int p = r ^ 1;
    if (p < N) {
      std::vector<double> s(M), d(M, -1.0);
      for (size_t i = 0; i < M; ++i) s[i] = r * 1e7 + i + rep;
      ncclGroupStart();
      ncclSend(s.data(), M, ncclFloat64, p, c, nullptr);
      ncclRecv(d.data(), M, ncclFloat64, p, c, nullptr);
      ncclGroupEnd();
      for (size_t i = 0; i < M; ++i) bad += d[i] != p * 1e7 + i + rep;
    }
  }
  ncclCommDestroy(c);
  return bad != 0;
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 4;
  ncclUniqueId id;
  ncclGetUniqueId(&id);
  std::vector<pid_t> kids;
  for (int r = 1; r < N; ++r) {
    pid_t k = fork();
    if (k == 0) _exit(run_rank(id, N, r));
    kids.push_back(k);
  }
  int fails = run_rank(id, N, 0);
  for (pid_t k : kids) {
    int st = 0;
    waitpid(k, &st, 0);
    fails += !(WIFEXITED(st) && WEXITSTATUS(st) == 0);
  }
  printf("%s (%d ranks)\n", fails ? "FAIL" : "OK", N);
  return fails != 0;
}
