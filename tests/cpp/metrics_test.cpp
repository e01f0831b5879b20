// metrics_test -- CPU driver of the C++ quality harness (espn::gpu::mrr_at_k /
// recall_at_k / load_qrels, include/espn_b200.hpp).  Reads a qrels file and a
// results file (`query_id doc_id...` per line, in rank order) and prints
// `mrr@k recall@k` for each k on the command line; `error <class>` on throw.
// Run by tests/test_quality.py, which checks it against the Python mirror.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>

#include "espn_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  try {
    espn::Qrels qrels = espn::gpu::load_qrels(std::filesystem::path(argv[1]));
    espn::ResultsByQuery res;
    std::ifstream f(argv[2]);
    std::string line;
    while (std::getline(f, line)) {
      std::istringstream ls(line);
      unsigned qid, did;
      if (!(ls >> qid)) continue;
      auto& rl = res[qid];
      float s = 1e6f;
      while (ls >> did) rl.entries.push_back(espn::ScoredDoc{did, s -= 1.f});
    }
    for (int i = 3; i < argc; ++i) {
      const int k = std::atoi(argv[i]);
      std::printf("%.17g %.17g\n", espn::gpu::mrr_at_k(res, qrels, k), espn::gpu::recall_at_k(res, qrels, k));
    }
  } catch (const espn::FormatError& e) {
    std::printf("error FormatError\n");
  } catch (const espn::IoError& e) {
    std::printf("error IoError\n");
  } catch (const espn::InvalidInputError& e) {
    std::printf("error InvalidInputError\n");
  }
  return 0;
}
