// Host half of the bottom-up person assembly (paf.cu scores the candidates):
// per limb type, valid candidates in descending score (ties: lower a, then
// lower b) are taken greedily while both peaks are unused, at most
// min(#A, #B) of them; each taken limb joins the person that already holds one
// of its peaks, merges two people that hold one each (when their parts do not
// overlap), or starts a new person (limb types < new_row_limbs only). People
// with >= 4 parts and total score / parts >= 0.4 are reported.
#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.hpp"

namespace avec {

namespace {

struct Conn {
  float score;
  int a, b;
};

struct Person {
  std::vector<int> part;  // peak index per part, -1 = none
  float score = 0.f;      // peaks' scores + limb scores
  float count = 0.f;      // parts found
};

}  // namespace

int assemble_people(const int* counts, const float* peaks, int n_parts, int max_peaks, const float* cand,
                    const int* limb_parts, int n_limbs, int new_row_limbs, int max_people, int* people,
                    float* people_score) {
  std::vector<Person> rows;
  std::vector<Conn> conns;
  std::vector<char> used_a(max_peaks), used_b(max_peaks);
  auto peak_score = [&](int part, int i) { return peaks[(static_cast<size_t>(part) * max_peaks + i) * 5 + 4]; };
  for (int l = 0; l < n_limbs; ++l) {
    const int pa = limb_parts[2 * l], pb = limb_parts[2 * l + 1];
    if (pa < 0 || pa >= n_parts || pb < 0 || pb >= n_parts) fail(AVEC_ERR_INVALID_ARGUMENT, "limb part index");
    const int na = std::min(counts[pa], max_peaks), nb = std::min(counts[pb], max_peaks);
    conns.clear();
    for (int a = 0; a < na; ++a)
      for (int b = 0; b < nb; ++b) {
        const float* c = cand + ((static_cast<size_t>(l) * max_peaks + a) * max_peaks + b) * 2;
        if (c[1] != 0.0f) conns.push_back({c[0], a, b});
      }
    std::sort(conns.begin(), conns.end(), [](const Conn& p, const Conn& q) {
      if (p.score != q.score) return p.score > q.score;
      return p.a != q.a ? p.a < q.a : p.b < q.b;
    });
    std::fill(used_a.begin(), used_a.end(), 0);
    std::fill(used_b.begin(), used_b.end(), 0);
    const int limit = std::min(na, nb);
    int taken = 0;
    for (const Conn& cn : conns) {
      if (taken >= limit) break;
      if (used_a[cn.a] || used_b[cn.b]) continue;
      used_a[cn.a] = used_b[cn.b] = 1;
      ++taken;
      int found = 0, idx[2] = {-1, -1};
      for (size_t j = 0; j < rows.size() && found < 2; ++j)
        if (rows[j].part[pa] == cn.a || rows[j].part[pb] == cn.b) idx[found++] = int(j);
      auto extend = [&](Person& r) {
        if (r.part[pb] != cn.b) {
          r.part[pb] = cn.b;
          r.count += 1.0f;
          r.score += peak_score(pb, cn.b) + cn.score;
        }
      };
      if (found == 1) {
        extend(rows[idx[0]]);
      } else if (found == 2) {
        Person& r1 = rows[idx[0]];
        const Person& r2 = rows[idx[1]];
        bool overlap = false;
        for (int p = 0; p < n_parts; ++p) overlap = overlap || (r1.part[p] >= 0 && r2.part[p] >= 0);
        if (!overlap) {
          for (int p = 0; p < n_parts; ++p)
            if (r2.part[p] >= 0) r1.part[p] = r2.part[p];
          r1.score += r2.score + cn.score;
          r1.count += r2.count;
          rows.erase(rows.begin() + idx[1]);
        } else {
          extend(r1);
        }
      } else if (l < new_row_limbs) {
        Person r;
        r.part.assign(n_parts, -1);
        r.part[pa] = cn.a;
        r.part[pb] = cn.b;
        r.score = peak_score(pa, cn.a) + peak_score(pb, cn.b) + cn.score;
        r.count = 2.0f;
        rows.push_back(std::move(r));
      }
    }
  }
  int out = 0;
  for (const Person& r : rows) {
    if (out >= max_people) break;
    if (r.count < 4.0f || r.score / r.count < 0.4f) continue;
    std::memcpy(people + static_cast<size_t>(out) * n_parts, r.part.data(), sizeof(int) * n_parts);
    people_score[2 * out] = r.score;
    people_score[2 * out + 1] = r.count;
    ++out;
  }
  return out;
}

}  // namespace avec
