// FTT1 transfer-table ingest for the halo plan:
// reader / writer of the reference's binary transfer-table format
// (proj/include/bsfv/tables.hpp:62-71) and its send/recv
// matching check (tables.cpp:185-235), exposed through the C-ABI.  The face
// entries of a rank's table drive sip_set_halo_tables (sip_api.cu), which
// allows arbitrary decompositions and periodic wraps (transfers.cpp:15-25).
//
// Entry rows are int[12]: dir, kind, face, peer, owner, neighbor, ilo, ihi,
// jlo, jhi, klo, khi -- the file's 40-byte record in field order.  Error
// texts and byte offsets follow the reference reader / validator so a
// caller's diagnostics do not change.
#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sip_c.h"
#include "sip_internal.h"

namespace sipb {
namespace {

constexpr int kRow = 12;

struct FormatFail {
  std::string what;
  size_t offset;
};

// little-endian cursor over an in-memory FTT1 image
class Cursor {
 public:
  Cursor(const unsigned char* p, size_t n) : p_(p), n_(n) {}
  size_t at() const { return at_; }
  unsigned u8(const char* field) {
    need(1, field);
    return p_[at_++];
  }
  uint32_t u32(const char* field) {
    need(4, field);
    uint32_t v = 0;
    for (int b = 3; b >= 0; --b) v = (v << 8) | p_[at_ + b];
    at_ += 4;
    return v;
  }

 private:
  void need(size_t k, const char* field) {
    if (at_ + k > n_) {
      // the reference reads byte-wise from a stream: a short read of a
      // u32 fails at the offset where the field started
      throw FormatFail{std::string("transfer table file truncated reading ") + field, at_};
    }
  }
  const unsigned char* p_;
  size_t n_, at_ = 0;
};

void put32(std::vector<unsigned char>& out, uint32_t v) {
  for (int b = 0; b < 4; ++b) out.push_back(static_cast<unsigned char>((v >> (8 * b)) & 0xFFu));
}

std::string box_str(const int* r) {  // Box::str(): "[ilo..ihi,jlo..jhi,klo..khi]"
  return "[" + std::to_string(r[6]) + ".." + std::to_string(r[7]) + "," + std::to_string(r[8]) +
         ".." + std::to_string(r[9]) + "," + std::to_string(r[10]) + ".." + std::to_string(r[11]) + "]";
}

long long box_cells(const int* r) {
  long long c = 1;
  for (int a = 0; a < 3; ++a) {
    const long long e = (long long)r[7 + 2 * a] - r[6 + 2 * a] + 1;
    c *= e > 0 ? e : 0;
  }
  return c;
}

}  // namespace

// Parse an FTT1 image: per-rank entry rows.
bool ftt1_parse(const unsigned char* buf, size_t len, std::vector<std::vector<std::array<int, 12>>>& out,
                std::string& err, long long& err_offset) {
  out.clear();
  try {
    Cursor c(buf, len);
    static const char magic[4] = {'F', 'T', 'T', '1'};
    for (int i = 0; i < 4; ++i) c.u8("magic");
    if (std::memcmp(buf, magic, 4) != 0) throw FormatFail{"bad magic, expected \"FTT1\"", 0};
    const uint32_t version = c.u32("version");
    if (version != 1) throw FormatFail{"unsupported format version " + std::to_string(version), 4};
    const uint32_t ranks = c.u32("rank count");
    c.u32("reserved");
    for (uint32_t r = 0; r < ranks; ++r) {
      const uint32_t n = c.u32("entry count");
      out.emplace_back();
      for (uint32_t k = 0; k < n; ++k) {
        const size_t off = c.at();
        std::array<int, 12> row{};
        const unsigned dir = c.u8("direction"), kind = c.u8("kind"), face = c.u8("face id");
        c.u8("pad");
        if (dir > 2) throw FormatFail{"invalid direction " + std::to_string(dir), off};
        if (kind > 2) throw FormatFail{"invalid patch kind " + std::to_string(kind), off + 1};
        if (face > 5) throw FormatFail{"invalid face id " + std::to_string(face), off + 2};
        row[0] = (int)dir;
        row[1] = (int)kind;
        row[2] = (int)face;
        row[3] = (int)c.u32("peer rank");
        row[4] = (int)c.u32("owner block");
        row[5] = (int)c.u32("neighbor block");
        for (int a = 0; a < 6; ++a) row[6 + a] = (int)c.u32("bounds");
        out.back().push_back(row);
      }
    }
  } catch (const FormatFail& f) {
    err = f.what + " (at byte offset " + std::to_string(f.offset) + ")";
    err_offset = (long long)f.offset;
    return false;
  }
  return true;
}

// tables.cpp:185-235 semantics: the k-th send A->B pairs with the k-th recv
// on B from A (same kind, swapped blocks, same cell count); no self sends,
// local entries name their own rank, no orphan recvs.
bool ftt1_validate(const std::vector<std::vector<std::array<int, 12>>>& t, std::string& err) {
  std::map<std::pair<int, int>, std::vector<const int*>> snd, rcv;
  for (int r = 0; r < (int)t.size(); ++r)
    for (const auto& row : t[r]) {
      const int peer = row[3];
      if (row[0] == 1) {
        if (peer == r) {
          err = "rank " + std::to_string(r) + " has a send entry targeting itself";
          return false;
        }
        snd[{r, peer}].push_back(row.data());
      } else if (row[0] == 2) {
        rcv[{peer, r}].push_back(row.data());
      } else if (peer != r) {
        err = "rank " + std::to_string(r) + " has a local entry with peer " + std::to_string(peer);
        return false;
      }
    }
  for (const auto& s : snd) {
    const auto it = rcv.find(s.first);
    const size_t nr = it == rcv.end() ? 0 : it->second.size();
    const std::string pair = std::to_string(s.first.first) + "->" + std::to_string(s.first.second);
    if (nr != s.second.size()) {
      err = "pair " + pair + " has " + std::to_string(s.second.size()) + " sends but " +
            std::to_string(nr) + " recvs";
      return false;
    }
    for (size_t k = 0; k < nr; ++k) {
      const int* a = s.second[k];
      const int* b = it->second[k];
      if (a[1] != b[1] || a[4] != b[5] || a[5] != b[4] || box_cells(a) != box_cells(b)) {
        err = "pair " + pair + " entry " + std::to_string(k) + " mismatched: send " + box_str(a) +
              " blocks " + std::to_string((unsigned)a[4]) + "/" + std::to_string((unsigned)a[5]) +
              " vs recv " + box_str(b);
        return false;
      }
    }
  }
  for (const auto& r : rcv)
    if (snd.find(r.first) == snd.end()) {
      err = "pair " + std::to_string(r.first.first) + "->" + std::to_string(r.first.second) +
            " has " + std::to_string(r.second.size()) + " recvs with no matching sends";
      return false;
    }
  return true;
}

static void rows_of(int nranks, const int* counts, const int* entries,
                    std::vector<std::vector<std::array<int, 12>>>& t) {
  t.assign(nranks, {});
  long long at = 0;
  for (int r = 0; r < nranks; ++r)
    for (int k = 0; k < counts[r]; ++k, ++at) {
      std::array<int, 12> row;
      for (int f = 0; f < kRow; ++f) row[f] = entries[at * kRow + f];
      t[r].push_back(row);
    }
}

}  // namespace sipb

using namespace sipb;

extern "C" {

int sip_ftt1_read(const void* buf, size_t len, int* nranks, int* counts, int* entries,
                  long long cap_entries, long long* total, long long* err_offset) {
  if (!buf || !nranks || !total) return SIP_ERR_MISUSE;
  std::vector<std::vector<std::array<int, 12>>> t;
  std::string err;
  long long off = -1;
  if (!ftt1_parse(static_cast<const unsigned char*>(buf), len, t, err, off)) {
    set_thread_error(err);
    if (err_offset) *err_offset = off;
    return SIP_ERR_FORMAT;
  }
  *nranks = (int)t.size();
  long long n = 0;
  for (const auto& r : t) n += (long long)r.size();
  *total = n;
  if (!counts || !entries) return SIP_OK;  // size query
  if (cap_entries < n) {
    set_thread_error("sip_ftt1_read: entry buffer too small");
    return SIP_ERR_MISUSE;
  }
  long long at = 0;
  for (size_t r = 0; r < t.size(); ++r) {
    counts[r] = (int)t[r].size();
    for (const auto& row : t[r]) {
      for (int f = 0; f < kRow; ++f) entries[at * kRow + f] = row[f];
      ++at;
    }
  }
  return SIP_OK;
}

int sip_ftt1_write(int nranks, const int* counts, const int* entries, void* buf, size_t cap,
                   size_t* len) {
  if (nranks < 0 || (nranks > 0 && (!counts || !entries)) || !len) return SIP_ERR_MISUSE;
  std::vector<unsigned char> out = {'F', 'T', 'T', '1'};
  put32(out, 1);
  put32(out, (uint32_t)nranks);
  put32(out, 0);
  long long at = 0;
  for (int r = 0; r < nranks; ++r) {
    put32(out, (uint32_t)counts[r]);
    for (int k = 0; k < counts[r]; ++k, ++at) {
      const int* e = entries + at * kRow;
      out.push_back((unsigned char)e[0]);
      out.push_back((unsigned char)e[1]);
      out.push_back((unsigned char)e[2]);
      out.push_back(0);
      for (int f = 3; f < kRow; ++f) put32(out, (uint32_t)e[f]);
    }
  }
  *len = out.size();
  if (!buf) return SIP_OK;  // size query
  if (cap < out.size()) {
    set_thread_error("sip_ftt1_write: buffer too small");
    return SIP_ERR_MISUSE;
  }
  std::memcpy(buf, out.data(), out.size());
  return SIP_OK;
}

int sip_ftt1_validate(int nranks, const int* counts, const int* entries) {
  if (nranks < 0 || (nranks > 0 && (!counts || !entries))) return SIP_ERR_MISUSE;
  std::vector<std::vector<std::array<int, 12>>> t;
  rows_of(nranks, counts, entries, t);
  std::string err;
  if (!ftt1_validate(t, err)) {
    set_thread_error(err);
    return SIP_ERR_PROTOCOL;
  }
  return SIP_OK;
}

}  // extern "C"
