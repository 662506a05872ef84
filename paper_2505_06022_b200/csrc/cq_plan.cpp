// Native command planner: region algebra + generate_commands in C++.
//
// Produces exactly the Plan of the Python planner (paper_2505_06022_b200/
// scheduler.py), which itself reproduces the reference's
// (pkg/src/clusterq/scheduler.py:224-369) command for command -- ids, deps,
// push sources, versions and the canonical box decomposition of every region
// (region.py:113-170: axis-0-first subtraction, per-axis greedy merge to a
// fixpoint, sort by (mins, maxs)).  Frequencies are attached by the Python
// side (exact-rational selection, energy.py:93-106).
//
// Wire format (int64 words) -- program in:
//   [n_buffers] { dims, extent[dims], initialized, element_bytes }*
//   [n_tasks]   { dims, range_hi[dims], n_pred, pred_task_index*, n_acc,
//                 { buffer, mode(0 read / 1 write), mapper, params... }* }*
//   mapper 0 one_to_one; 1 neighborhood radii[buffer dims]; 2 all;
//          3 slice axis; 4 fixed n_boxes {lo[d], hi[d]}*
// plan out:
//   [n_commands] { kind(0 exec / 1 push / 2 await), n_deps, deps*, fields }*
//   exec : task_index, node, chunk lo[d], hi[d], n_reads {acc, region}*,
//          n_writes {acc, region, version}*
//   push : src, dst, buffer, version, region
//   await: dst, buffer, version, push_id, region
//   then per buffer: n_entries { version, n_holders, holder*, region }*
//   region = n_boxes { lo[d], hi[d] }*
#include <stdint.h>

#include <algorithm>
#include <array>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "../../include/cq.h"

namespace cq {
void set_error(const char* fmt, ...);
}

namespace {

constexpr int D = 3;
struct Box {
  std::array<int64_t, D> lo{}, hi{};
  bool operator<(const Box& o) const {
    if (lo != o.lo) return lo < o.lo;
    return hi < o.hi;
  }
  bool operator==(const Box& o) const { return lo == o.lo && hi == o.hi; }
};

struct Region {
  int dims = 1;
  std::vector<Box> boxes;  // canonical
  bool empty() const { return boxes.empty(); }
};

inline bool box_empty(const Box& b, int d) {
  for (int k = 0; k < d; ++k)
    if (b.lo[k] >= b.hi[k]) return true;
  return false;
}

inline bool overlap(const Box& a, const Box& b, int d, Box* out) {
  Box r;
  for (int k = 0; k < d; ++k) {
    r.lo[k] = std::max(a.lo[k], b.lo[k]);
    r.hi[k] = std::min(a.hi[k], b.hi[k]);
    if (r.lo[k] >= r.hi[k]) return false;
  }
  if (out) *out = r;
  return true;
}

// a \ b, axis by axis (dimension 0 first), earlier axes clamped to a & b
void subtract(const Box& a, const Box& b, int d, std::vector<Box>& out) {
  Box cut;
  if (!overlap(a, b, d, &cut)) {
    if (!box_empty(a, d)) out.push_back(a);
    return;
  }
  Box core = a;
  for (int k = 0; k < d; ++k) {
    if (core.lo[k] < cut.lo[k]) {
      Box p = core;
      p.hi[k] = cut.lo[k];
      out.push_back(p);
    }
    if (cut.hi[k] < core.hi[k]) {
      Box p = core;
      p.lo[k] = cut.hi[k];
      out.push_back(p);
    }
    core.lo[k] = cut.lo[k];
    core.hi[k] = cut.hi[k];
  }
}

std::vector<Box> subtract_all(std::vector<Box> pieces, const std::vector<Box>& cutters, int d) {
  for (const Box& c : cutters) {
    std::vector<Box> nxt;
    nxt.reserve(pieces.size() + 4);
    for (const Box& p : pieces) {
      if (!overlap(p, c, d, nullptr)) nxt.push_back(p);
      else subtract(p, c, d, nxt);
    }
    pieces.swap(nxt);
    if (pieces.empty()) break;
  }
  return pieces;
}

// one greedy merge pass along `axis`; groups keyed by the other axes' bounds
// (visited in sorted key order, as the Python dict-of-sorted-keys does)
bool merge_pass(std::vector<Box>& boxes, int axis, int d) {
  typedef std::pair<std::vector<int64_t>, std::vector<int64_t>> Key;
  std::map<Key, std::vector<Box>> groups;
  for (const Box& b : boxes) {
    Key key;
    for (int k = 0; k < d; ++k)
      if (k != axis) {
        key.first.push_back(b.lo[k]);
        key.second.push_back(b.hi[k]);
      }
    groups[key].push_back(b);
  }
  std::vector<Box> out;
  out.reserve(boxes.size());
  bool merged = false;
  for (auto& kv : groups) {
    auto& run = kv.second;
    if (run.size() > 1)
      std::sort(run.begin(), run.end(), [axis](const Box& x, const Box& y) { return x.lo[axis] < y.lo[axis]; });
    Box cur = run[0];
    for (size_t i = 1; i < run.size(); ++i) {
      if (cur.hi[axis] == run[i].lo[axis]) {
        cur.hi[axis] = run[i].hi[axis];
        merged = true;
      } else {
        out.push_back(cur);
        cur = run[i];
      }
    }
    out.push_back(cur);
  }
  boxes.swap(out);
  return merged;
}

Region canonical(int d, std::vector<Box> boxes) {
  Region r;
  r.dims = d;
  for (const Box& b : boxes)
    if (!box_empty(b, d)) r.boxes.push_back(b);
  if (r.boxes.size() > 1) {
    for (;;) {
      bool changed = false;
      for (int axis = 0; axis < d; ++axis) changed = merge_pass(r.boxes, axis, d) || changed;
      if (!changed) break;
    }
    std::sort(r.boxes.begin(), r.boxes.end());
  }
  return r;
}

Region from_box(const Box& b, int d) {
  Region r;
  r.dims = d;
  if (!box_empty(b, d)) r.boxes.push_back(b);
  return r;
}

Region runion(const Region& a, const Region& b) {
  if (b.empty()) return a;
  if (a.empty()) return b;
  std::vector<Box> extra;
  for (const Box& x : b.boxes) {
    auto p = subtract_all({x}, a.boxes, a.dims);
    extra.insert(extra.end(), p.begin(), p.end());
  }
  if (extra.empty()) return a;
  std::vector<Box> all = a.boxes;
  all.insert(all.end(), extra.begin(), extra.end());
  return canonical(a.dims, all);
}

Region rintersect(const Region& a, const Region& b) {
  std::vector<Box> hits;
  for (const Box& x : a.boxes)
    for (const Box& y : b.boxes) {
      Box c;
      if (overlap(x, y, a.dims, &c)) hits.push_back(c);
    }
  return canonical(a.dims, hits);
}

Region rdifference(const Region& a, const Region& b) {
  if (a.empty() || b.empty()) return a;
  return canonical(a.dims, subtract_all(a.boxes, b.boxes, a.dims));
}

bool roverlaps(const Region& a, const Region& b) {
  for (const Box& x : a.boxes)
    for (const Box& y : b.boxes)
      if (overlap(x, y, a.dims, nullptr)) return true;
  return false;
}

int64_t rvolume(const Region& a) {
  int64_t v = 0;
  for (const Box& b : a.boxes) {
    int64_t n = 1;
    for (int k = 0; k < a.dims; ++k) n *= b.hi[k] - b.lo[k];
    v += n;
  }
  return v;
}

// ---------------------------------------------------------------- model
struct Buffer {
  int dims;
  Box extent;
  bool initialized;
  int64_t ebytes;
};

struct Mapper {
  int kind = 0;
  std::array<int64_t, D> radii{};
  int axis = 0;
  Region fixed;
};

struct Acc {
  int buffer;
  int mode;  // 0 read, 1 write
  Mapper m;
};

struct Task {
  int dims;
  Box range;
  std::vector<int> preds;
  std::vector<Acc> accs;
};

Region clip(const Box& b, const Box& extent, int d) {
  Box c;
  if (!overlap(b, extent, d, &c)) return Region{d, {}};
  return from_box(c, d);
}

// mapper image of `chunk` (model.py:135-231)
Region map_chunk(const Mapper& m, const Box& chunk, const Buffer& buf) {
  int d = buf.dims;
  switch (m.kind) {
    case 0:
      return clip(chunk, buf.extent, d);
    case 1: {
      Box g = chunk;
      for (int k = 0; k < d; ++k) {
        g.lo[k] -= m.radii[k];
        g.hi[k] += m.radii[k];
      }
      return clip(g, buf.extent, d);
    }
    case 2:
      return from_box(buf.extent, d);
    case 3: {
      Box g = chunk;
      g.lo[m.axis] = buf.extent.lo[m.axis];
      g.hi[m.axis] = buf.extent.hi[m.axis];
      return clip(g, buf.extent, d);
    }
    default:
      return rintersect(m.fixed, from_box(buf.extent, d));
  }
}

struct Piece {
  Region region;
  int64_t version;
  std::map<int, int64_t> holders;  // node -> producer (-1: host data)
};

struct Cmd {
  int kind;
  int64_t id;
  std::vector<int64_t> deps;
  // exec
  int task = -1, node = -1;
  Box chunk;
  std::vector<std::pair<int, Region>> reads;
  std::vector<std::tuple<int, Region, int64_t>> writes;
  // push / await
  int src = -1, dst = -1, buffer = -1;
  int64_t version = 0, push_id = -1;
  Region region;
};

struct Reader {
  const int64_t* p;
  const int64_t* end;
  int64_t next() {
    if (p >= end) throw std::string("program stream truncated");
    return *p++;
  }
};

void put_region(std::vector<int64_t>& o, const Region& r, int d) {
  o.push_back((int64_t)r.boxes.size());
  for (const Box& b : r.boxes) {
    for (int k = 0; k < d; ++k) o.push_back(b.lo[k]);
    for (int k = 0; k < d; ++k) o.push_back(b.hi[k]);
  }
}

std::vector<int64_t> plan(const int64_t* prog, int64_t len, int nodes) {
  Reader rd{prog, prog + len};
  std::vector<Buffer> bufs(rd.next());
  for (auto& b : bufs) {
    b.dims = (int)rd.next();
    for (int k = 0; k < b.dims; ++k) b.extent.hi[k] = rd.next();
    b.initialized = rd.next() != 0;
    b.ebytes = rd.next();
  }
  std::vector<Task> tasks(rd.next());
  for (auto& t : tasks) {
    t.dims = (int)rd.next();
    for (int k = 0; k < t.dims; ++k) t.range.hi[k] = rd.next();
    int np = (int)rd.next();
    for (int i = 0; i < np; ++i) t.preds.push_back((int)rd.next());
    int na = (int)rd.next();
    for (int i = 0; i < na; ++i) {
      Acc a;
      a.buffer = (int)rd.next();
      a.mode = (int)rd.next();
      a.m.kind = (int)rd.next();
      int bd = bufs[a.buffer].dims;
      if (a.m.kind == 1)
        for (int k = 0; k < bd; ++k) a.m.radii[k] = rd.next();
      else if (a.m.kind == 3)
        a.m.axis = (int)rd.next();
      else if (a.m.kind == 4) {
        int nb = (int)rd.next();
        std::vector<Box> bx(nb);
        for (auto& b : bx) {
          for (int k = 0; k < bd; ++k) b.lo[k] = rd.next();
          for (int k = 0; k < bd; ++k) b.hi[k] = rd.next();
        }
        // the Python Fixed region is already canonical; rebuild through the
        // constructor semantics (disjoint pieces in order, then canonical)
        std::vector<Box> acc;
        for (const Box& b : bx) {
          if (box_empty(b, bd)) continue;
          auto p = subtract_all({b}, acc, bd);
          acc.insert(acc.end(), p.begin(), p.end());
        }
        a.m.fixed = canonical(bd, acc);
      }
      t.accs.push_back(a);
    }
  }

  // region map table (scheduler.py:120-184)
  std::vector<std::vector<Piece>> table(bufs.size());
  std::vector<int64_t> vcount(bufs.size());
  for (size_t b = 0; b < bufs.size(); ++b) {
    if (bufs[b].initialized) {
      table[b].push_back(Piece{from_box(bufs[b].extent, bufs[b].dims), 1, {{0, -1}}});
      vcount[b] = 1;
    }
  }
  auto resident = [&](int b, int node) {
    Region acc{bufs[b].dims, {}};
    for (const Piece& p : table[b])
      if (p.holders.count(node)) acc = runion(acc, p.region);
    return acc;
  };
  auto covered = [&](int b) {
    Region acc{bufs[b].dims, {}};
    for (const Piece& p : table[b]) acc = runion(acc, p.region);
    return acc;
  };

  std::vector<Cmd> cmds;
  std::vector<std::vector<int64_t>> execs_of(tasks.size());
  for (size_t ti = 0; ti < tasks.size(); ++ti) {
    const Task& t = tasks[ti];
    std::set<int64_t> pred_execs;
    for (int p : t.preds)
      for (int64_t e : execs_of[p]) pred_execs.insert(e);
    std::vector<int> written;
    std::map<int, int64_t> new_version;
    for (const Acc& a : t.accs)
      if (a.mode == 1 && !new_version.count(a.buffer)) {
        new_version[a.buffer] = vcount[a.buffer] + 1;
        written.push_back(a.buffer);
      }
    // split_task (scheduler.py:37-53)
    int64_t extent0 = t.range.hi[0] - t.range.lo[0];
    int64_t base = extent0 / nodes, extra = extent0 % nodes;
    std::vector<int64_t> pushes, execs;
    struct Gain {
      int b;
      Region r;
      int node;
      int64_t ap;
    };
    std::vector<Gain> gains;
    int64_t start = t.range.lo[0];
    for (int node = 0; node < std::min<int64_t>(nodes, extent0); ++node) {
      int64_t size = base + (node < extra ? 1 : 0);
      Box chunk = t.range;
      chunk.lo[0] = start;
      chunk.hi[0] = start + size;
      start += size;
      std::vector<std::pair<int, Region>> reads;
      std::vector<std::pair<int, Region>> need;  // insertion-ordered per buffer
      for (int ai = 0; ai < (int)t.accs.size(); ++ai) {
        const Acc& a = t.accs[ai];
        if (a.mode != 0) continue;
        Region img = map_chunk(a.m, chunk, bufs[a.buffer]);
        reads.push_back({ai, img});
        auto it = std::find_if(need.begin(), need.end(), [&](auto& x) { return x.first == a.buffer; });
        if (it == need.end()) need.push_back({a.buffer, img});
        else it->second = runion(it->second, img);
      }
      std::vector<int64_t> awaited;
      for (auto& nb : need) {
        int b = nb.first;
        Region gap = rdifference(nb.second, resident(b, node));
        if (gap.empty()) continue;
        Region never = rdifference(gap, covered(b));
        if (!never.empty()) throw std::string("uninitialized read");
        for (const Piece& pc : table[b]) {
          Region part = rintersect(pc.region, gap);
          if (part.empty()) continue;
          int src = pc.holders.begin()->first;
          int64_t producer = pc.holders.begin()->second;
          Cmd push;
          push.kind = 1;
          push.id = (int64_t)cmds.size();
          if (producer >= 0) push.deps.push_back(producer);
          push.src = src;
          push.dst = node;
          push.buffer = b;
          push.region = part;
          push.version = pc.version;
          cmds.push_back(push);
          pushes.push_back(push.id);
          Cmd ap;
          ap.kind = 2;
          ap.id = (int64_t)cmds.size();
          ap.deps.push_back(push.id);
          ap.dst = node;
          ap.buffer = b;
          ap.region = part;
          ap.version = pc.version;
          ap.push_id = push.id;
          cmds.push_back(ap);
          awaited.push_back(ap.id);
          gains.push_back({b, part, node, ap.id});
        }
      }
      Cmd exe;
      exe.kind = 0;
      exe.id = (int64_t)cmds.size();
      std::set<int64_t> deps(pred_execs);
      deps.insert(awaited.begin(), awaited.end());
      exe.deps.assign(deps.begin(), deps.end());
      exe.task = (int)ti;
      exe.node = node;
      exe.chunk = chunk;
      exe.reads = reads;
      for (int ai = 0; ai < (int)t.accs.size(); ++ai) {
        const Acc& a = t.accs[ai];
        if (a.mode != 1) continue;
        exe.writes.emplace_back(ai, map_chunk(a.m, chunk, bufs[a.buffer]), new_version[a.buffer]);
      }
      cmds.push_back(exe);
      execs.push_back(exe.id);
    }
    // in-place hazards (scheduler.py:336-348)
    for (int64_t eid : execs) {
      Cmd& exe = cmds[eid];
      std::set<int64_t> extra_deps;
      for (int64_t pid : pushes) {
        const Cmd& p = cmds[pid];
        if (p.src != exe.node) continue;
        for (auto& w : exe.writes) {
          if (t.accs[std::get<0>(w)].buffer == p.buffer && roverlaps(std::get<1>(w), p.region)) {
            extra_deps.insert(pid);
            break;
          }
        }
      }
      if (!extra_deps.empty()) {
        extra_deps.insert(exe.deps.begin(), exe.deps.end());
        exe.deps.assign(extra_deps.begin(), extra_deps.end());
      }
    }
    for (auto& g : gains) {
      std::vector<Piece> upd;
      for (const Piece& pc : table[g.b]) {
        Region shared = rintersect(pc.region, g.r);
        if (shared.empty()) {
          upd.push_back(pc);
          continue;
        }
        Region rest = rdifference(pc.region, shared);
        if (!rest.empty()) upd.push_back(Piece{rest, pc.version, pc.holders});
        Piece np{shared, pc.version, pc.holders};
        np.holders[g.node] = g.ap;
        upd.push_back(np);
      }
      table[g.b].swap(upd);
    }
    for (int b : written) {
      int64_t version = ++vcount[b];
      for (int64_t eid : execs) {
        const Cmd& exe = cmds[eid];
        for (auto& w : exe.writes) {
          if (t.accs[std::get<0>(w)].buffer != b) continue;
          const Region& reg = std::get<1>(w);
          std::vector<Piece> upd;
          for (const Piece& pc : table[b]) {
            Region rest = rdifference(pc.region, reg);
            if (!rest.empty()) upd.push_back(Piece{rest, pc.version, pc.holders});
          }
          upd.push_back(Piece{reg, version, {{exe.node, exe.id}}});
          table[b].swap(upd);
        }
      }
    }
    execs_of[ti] = execs;
  }

  std::vector<int64_t> o;
  o.push_back((int64_t)cmds.size());
  for (const Cmd& c : cmds) {
    o.push_back(c.kind);
    o.push_back((int64_t)c.deps.size());
    o.insert(o.end(), c.deps.begin(), c.deps.end());
    if (c.kind == 0) {
      const Task& t = tasks[c.task];
      o.push_back(c.task);
      o.push_back(c.node);
      for (int k = 0; k < t.dims; ++k) o.push_back(c.chunk.lo[k]);
      for (int k = 0; k < t.dims; ++k) o.push_back(c.chunk.hi[k]);
      o.push_back((int64_t)c.reads.size());
      for (auto& r : c.reads) {
        o.push_back(r.first);
        put_region(o, r.second, bufs[t.accs[r.first].buffer].dims);
      }
      o.push_back((int64_t)c.writes.size());
      for (auto& w : c.writes) {
        o.push_back(std::get<0>(w));
        put_region(o, std::get<1>(w), bufs[t.accs[std::get<0>(w)].buffer].dims);
        o.push_back(std::get<2>(w));
      }
    } else if (c.kind == 1) {
      o.push_back(c.src);
      o.push_back(c.dst);
      o.push_back(c.buffer);
      o.push_back(c.version);
      put_region(o, c.region, bufs[c.buffer].dims);
    } else {
      o.push_back(c.dst);
      o.push_back(c.buffer);
      o.push_back(c.version);
      o.push_back(c.push_id);
      put_region(o, c.region, bufs[c.buffer].dims);
    }
  }
  for (size_t b = 0; b < bufs.size(); ++b) {
    o.push_back((int64_t)table[b].size());
    for (const Piece& pc : table[b]) {
      o.push_back(pc.version);
      o.push_back((int64_t)pc.holders.size());
      for (auto& h : pc.holders) o.push_back(h.first);
      put_region(o, pc.region, bufs[b].dims);
    }
  }
  return o;
}

}  // namespace

extern "C" {

int cq_plan_generate(const int64_t* program, int64_t length, int node_count, int64_t** out, int64_t* out_length) {
  if (node_count < 1) {
    cq::set_error("node count must be at least 1");
    return CQ_ERR_ARG;
  }
  try {
    std::vector<int64_t> o = plan(program, length, node_count);
    int64_t* buf = new int64_t[o.size()];
    std::copy(o.begin(), o.end(), buf);
    *out = buf;
    *out_length = (int64_t)o.size();
    return CQ_OK;
  } catch (const std::string& e) {
    cq::set_error("cq_plan_generate: %s", e.c_str());
    return CQ_ERR_ARG;
  }
}

int cq_plan_free(int64_t* out) {
  delete[] out;
  return CQ_OK;
}

}  // extern "C"
