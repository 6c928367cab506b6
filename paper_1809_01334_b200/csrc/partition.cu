// partition.cu -- exchange partners from the partition markers (SURVEY §8(f)
// NEXT(4); "Senders determine the receiving processes" /
// "Receivers determine the sending processes").
//
// Every rank knows the partition markers (tree and anchor of each rank's
// first leaf), the per-tree geometry and the camera, so
// the pairs (vforest rank p, writer q) that exchange ray segments follow
// without communication: a writer runs a virtual top-down traversal of every
// tree, splitting the marker range by nested binary searches, stops where a
// node's pixel-centre rectangle (SURVEY R6 on the node's camera-space
// Bernstein box) misses its tiles, and records the owner when the range holds
// a single rank.  The sender side evaluates the same
// relation for each writer (DESIGN D19), so both sides agree by construction
// and every rank posts exactly the matching sends and receives.  Node boxes
// are padded by RC_PARTNER_PAD world units so that they contain the device
// cull's leaf boxes despite rounding: every pair that carries a record is
// found (rc_composite_tiles checks this on every exchange).
//
// Host code: the traversal visits O(P x depth x 8) nodes per writer.
#include <stdint.h>
#include <string.h>

#include <vector>

#include "geom.cuh"

#define RC_PARTNER_PAD 1e-9

namespace {
using namespace rc;

struct Pos {   // SFC position: tree-major, Morton key of the level-18 anchor within a tree
  int32_t tree;
  uint64_t key;
};
inline bool operator<(const Pos& a, const Pos& b) { return a.tree < b.tree || (a.tree == b.tree && a.key < b.key); }
inline bool operator<=(const Pos& a, const Pos& b) { return !(b < a); }

uint64_t spread18(uint32_t v) {
  uint64_t x = v & 0x3FFFFu, r = 0;
  for (int b = 0; b < 18; ++b) r |= ((x >> b) & 1ull) << (3 * b);
  return r;
}
Pos pos_of(int32_t tree, const int32_t a[3]) {
  return Pos{tree, spread18((uint32_t)a[0]) | (spread18((uint32_t)a[1]) << 1) | (spread18((uint32_t)a[2]) << 2)};
}

struct Traversal {
  const rc_forest* f;
  std::vector<Pos> m;          // markers m_0..m_P
  int P;
  int tiles_x, tiles_y, tw, th;
  int writer;                  // the writer whose tiles are tested
  std::vector<uint8_t>* found; // [P]: ranks recorded as senders to `writer`

  bool nonempty(int p) const { return m[p] < m[p + 1]; }

  // node rectangle meets one of the writer's tiles
  bool meets_writer(const Rect16& r) const {
    const int tx0 = r.i0 / tw, tx1 = r.i1 / tw, ty0 = r.j0 / th, ty1 = r.j1 / th;
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx)
        if ((tx + ty) % P == writer) return true;   // tile owner map of rc_composite_tiles
    return false;
  }

  bool node_rect(int tree, const int32_t a[3], int level, Rect16& rc) const {
    const TreeConst& T = f->h_trees[tree];
    const double h = ldexp(1.0, -level);
    double t0[3];
    for (int k = 0; k < 3; ++k) t0[k] = ldexp((double)a[k], -RC_MAXLEVEL);
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    if (f->surface) {
      for (int q = 0; q < 4; ++q) {
        double X[3];
        patch_point(T.Bc, t0[0] + h * (q & 1), t0[1] + h * (q >> 1), X);
        for (int c = 0; c < 3; ++c) {
          lo[c] = fmin(lo[c], X[c]);
          hi[c] = fmax(hi[c], X[c]);
        }
      }
    } else if (f->R == 2) {
      element_aabb<2>(T.Bc, t0, h, lo, hi);
    } else {
      element_aabb<1>(T.Bc, t0, h, lo, hi);
    }
    for (int c = 0; c < 3; ++c) {
      lo[c] -= RC_PARTNER_PAD;
      hi[c] += RC_PARTNER_PAD;
    }
    return project_rect(f->cc, lo, hi, rc);
  }

  // ranks whose positions [m_p, m_{p+1}) meet [s, e), searched inside [lo, hi]
  void split(const Pos& s, const Pos& e, int lo, int hi, int& clo, int& chi) const {
    int a = lo, b = hi;   // last p in [lo, hi] with m_p <= s
    while (a < b) {
      const int mid = (a + b + 1) / 2;
      if (m[mid] <= s) a = mid;
      else b = mid - 1;
    }
    clo = a;
    a = lo, b = hi;       // last p in [lo, hi] with m_p < e
    while (a < b) {
      const int mid = (a + b + 1) / 2;
      if (m[mid] < e) a = mid;
      else b = mid - 1;
    }
    chi = a;
  }

  void recurse(int tree, const int32_t a[3], int level, int lo, int hi) {
    Rect16 rc;
    if (!node_rect(tree, a, level, rc) || !meets_writer(rc)) return;
    int only = -1, count = 0;
    for (int p = lo; p <= hi && count < 2; ++p)
      if (nonempty(p)) {
        only = p;
        ++count;
      }
    if (count == 0) return;
    if (count == 1) {
      (*found)[only] = 1;
      return;
    }
    if (level >= RC_MAXLEVEL) return;   // cannot happen for markers at leaf anchors
    const int32_t hh = 1 << (RC_MAXLEVEL - level - 1);
    const int nchild = f->surface ? 4 : 8;
    for (int c = 0; c < nchild; ++c) {
      const int32_t ca[3] = {a[0] + hh * (c & 1), a[1] + hh * ((c >> 1) & 1), a[2] + hh * ((c >> 2) & 1)};
      const Pos s = pos_of(tree, ca);
      // end of the child's positions: s + 8^(18-level-1)
      const uint64_t span = 1ull << (3 * (RC_MAXLEVEL - level - 1));
      Pos e{tree, s.key + span};
      if (s.key + span >= (1ull << (3 * RC_MAXLEVEL))) e = Pos{tree + 1, 0};
      int clo, chi;
      split(s, e, lo, hi, clo, chi);
      recurse(tree, ca, level + 1, clo, chi);
    }
  }

  void run() {
    const int32_t zero[3] = {0, 0, 0};
    for (int k = 0; k < f->K; ++k) {
      int clo, chi;
      split(Pos{k, 0}, Pos{k + 1, 0}, 0, P - 1, clo, chi);
      recurse(k, zero, 0, clo, chi);
    }
  }
};
}  // namespace

extern "C" rc_status rc_exchange_partners(rc_forest* f, const rc_tiling* t, const rc_marker* h_markers,
                                          uint8_t* h_send_to, uint8_t* h_recv_from) {
  RC_NVTX("rc_exchange_partners");
  if (!f || !t || !h_markers) return rc_fail(RC_ERR_INVALID_ARG, "rc_exchange_partners: null argument");
  if (!f->have_camera) return rc_fail(RC_ERR_STATE, "rc_exchange_partners before rc_camera_set");
  const int P = t->nranks;
  if (P < 1 || P > RC_MAX_RANKS || t->rank < 0 || t->rank >= P || t->tiles_x < 1 || t->tiles_y < 1 ||
      f->cc.W % t->tiles_x || f->cc.H % t->tiles_y)
    return rc_fail(RC_ERR_INVALID_ARG, "rc_exchange_partners: bad tiling");
  Traversal tr;
  tr.f = f;
  tr.P = P;
  tr.tiles_x = t->tiles_x;
  tr.tiles_y = t->tiles_y;
  tr.tw = f->cc.W / t->tiles_x;
  tr.th = f->cc.H / t->tiles_y;
  tr.m.resize(P + 1);
  for (int p = 0; p <= P; ++p) {
    const rc_marker& mk = h_markers[p];
    if (mk.tree < 0 || mk.tree > f->K) return rc_fail(RC_ERR_INVALID_ARG, "marker %d: bad tree %d", p, mk.tree);
    for (int k = 0; k < 3; ++k)
      if (mk.anchor[k] < 0 || mk.anchor[k] >= (1 << RC_MAXLEVEL))
        return rc_fail(RC_ERR_INVALID_ARG, "marker %d: anchor out of range", p);
    tr.m[p] = pos_of(mk.tree, mk.anchor);
    if (p > 0 && tr.m[p] < tr.m[p - 1]) return rc_fail(RC_ERR_INVALID_ARG, "markers not in SFC order at %d", p);
  }
  if (!(tr.m[P].tree == f->K && tr.m[P].key == 0))
    return rc_fail(RC_ERR_INVALID_ARG, "marker %d must be (num_trees, 0, 0, 0)", P);
  if (!(tr.m[0].tree == 0 && tr.m[0].key == 0)) return rc_fail(RC_ERR_INVALID_ARG, "marker 0 must be (0, 0, 0, 0)");
  std::vector<uint8_t> found(P, 0);
  tr.found = &found;
  if (h_recv_from) {   // receiver side: my senders
    tr.writer = t->rank;
    tr.run();
    memcpy(h_recv_from, found.data(), P);
  }
  if (h_send_to) {     // sender side: every writer whose traversal records me
    for (int q = 0; q < P; ++q) {
      std::fill(found.begin(), found.end(), 0);
      tr.writer = q;
      tr.run();
      h_send_to[q] = found[t->rank];
    }
  }
  return RC_OK;
}
