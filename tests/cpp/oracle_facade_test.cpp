// Own test (not a reference source): the Oracle cases of the reference's
// harness_test.cpp:88-180 restated on a box world built here (the harness's
// gen_scene / benchmark.hpp are not part of the facade), run through the C++
// facade's device-backed oracle_search and search.
#include <algorithm>
#include <cstdint>

#include <gtest/gtest.h>

#include "bnbloc/oracle.hpp"
#include "bnbloc/rng.hpp"
#include "bnbloc/search.hpp"

using namespace bnbloc;

namespace {

// floor 8x8 m plus two walls, points drawn uniformly on the surfaces
PointCloud box_world(std::uint64_t seed, int n) {
  Rng rng(seed);
  PointCloud c;
  for (int i = 0; i < n; ++i) {
    switch (i % 3) {
      case 0: c.points.push_back({rng.uniform(0, 8), rng.uniform(0, 8), 0.0}); break;
      case 1: c.points.push_back({rng.uniform(2, 5), 2.0, rng.uniform(0, 2.5)}); break;
      default: c.points.push_back({6.0, rng.uniform(3, 7), rng.uniform(0, 3)}); break;
    }
  }
  return c;
}

// scan = world samples seen from (tx, ty, 0): q = p - t
PointCloud scan_from(const PointCloud& w, double tx, double ty) {
  PointCloud s;
  for (const Point3& p : w.points) s.points.push_back({p.x - tx, p.y - ty, p.z});
  return s;
}

SearchConfig trans_only_cfg() {
  SearchConfig cfg;
  cfg.min_resolution = 1.0;
  cfg.max_level = 2;
  cfg.branch_mode = BranchMode::kTransOnly;
  cfg.roll_pitch_half_range = 0.0;
  cfg.yaw_min = -0.2;
  cfg.yaw_max = 0.2;
  cfg.score_threshold_fraction = 0.9;
  cfg.workers = 2;
  return cfg;
}

}  // namespace

TEST(Oracle, TinyMapMatchesTransOnlySearch) {
  for (std::uint64_t seed : {11ULL, 12ULL}) {
    const PointCloud map_cloud = box_world(seed, 6000);
    const PointCloud scan = scan_from(box_world(seed + 100, 900), 1.3, 0.7);
    SearchConfig cfg = trans_only_cfg();
    const MultiResVoxelMap map = MultiResVoxelMap::build(map_cloud, cfg.min_resolution, cfg.max_level, 0.01);
    const OracleResult oracle = oracle_search(map, scan, cfg);
    EXPECT_GT(oracle.leaf_count, 0u);
    EXPECT_FALSE(oracle.argmax_poses.empty());
    for (Strategy st : {Strategy::kDfs, Strategy::kBfs}) {
      cfg.strategy = st;
      const SearchResult r = search(map, scan, cfg);
      if (oracle.best_score >= r.score_threshold) {
        EXPECT_TRUE(r.matched);
        EXPECT_EQ(oracle.best_score, r.best_score);
      } else {
        EXPECT_FALSE(r.matched);
      }
    }
  }
}

TEST(Oracle, IndependentOfScanPointOrder) {
  const PointCloud map_cloud = box_world(5, 4000);
  const PointCloud scan = scan_from(box_world(105, 600), 0.4, 1.1);
  const SearchConfig cfg = trans_only_cfg();
  const MultiResVoxelMap map = MultiResVoxelMap::build(map_cloud, 1.0, 2, 0.01);
  const OracleResult a = oracle_search(map, scan, cfg);
  PointCloud reversed = scan;
  std::reverse(reversed.points.begin(), reversed.points.end());
  const OracleResult b = oracle_search(map, reversed, cfg);
  EXPECT_EQ(a.best_score, b.best_score);
  EXPECT_EQ(a.leaf_count, b.leaf_count);
  EXPECT_EQ(a.argmax_poses.size(), b.argmax_poses.size());
}

TEST(Oracle, GuardsAgainstHugeGrids) {
  PointCloud big;
  Rng rng(3);
  for (int i = 0; i < 2000; ++i)
    big.points.push_back({rng.uniform(0, 500), rng.uniform(0, 500), rng.uniform(0, 50)});
  const MultiResVoxelMap map = MultiResVoxelMap::build(big, 1.0, 2, 0.05);
  PointCloud scan;
  for (int i = 0; i < 100; ++i)
    scan.points.push_back({rng.uniform(-20, 20), rng.uniform(-20, 20), rng.uniform(-2, 2)});
  SearchConfig cfg;
  cfg.min_resolution = 1.0;
  cfg.max_level = 2;
  cfg.branch_mode = BranchMode::kTransOnly;
  EXPECT_THROW(oracle_search(map, scan, cfg), TooLargeError);
}
