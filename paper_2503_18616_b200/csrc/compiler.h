// compiler.h -- host scene compiler entry points (single-CTA programs and cluster parts).
#pragma once
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/tissuesim_b200.h"

namespace ts {

// One part of a cluster program: the CTA of rank `rank` (of K) of an environment's
// thread-block cluster owns the vertices with own[v] != 0 (updates and writes them back),
// handles the constraints touching its owned free vertices and the surface faces in `faces`,
// and reads a halo of other parts' vertices that their owners refresh over DSMEM.
struct PartSpec {
    int rank = 0, K = 1;
    std::vector<char> own;                 // [V]
    std::vector<int> faces;                // global face ids, ascending
    int force_B = 0, force_Vstore = 0, force_slot_cap = 0;
    // pass 2: for every vertex, the (rank, storage position) of each part holding it as halo,
    // and the (rank, storage position) of its owner
    const std::vector<std::vector<std::pair<int, int>>> *halo_of = nullptr;
    const std::vector<int> *owner_rank = nullptr, *owner_pos = nullptr;
};

int compile_program(const ts_scene_desc &d, const ts_layout_opts &o, std::vector<uint8_t> &blob,
                    ts_layout_info &info, std::string &err, const PartSpec *part = nullptr);

// K-part cluster program (TsClusterHeader + K part programs); K = 0 picks the smallest
// power of two whose parts fit one CTA each.
int compile_cluster(const ts_scene_desc &d, const ts_layout_opts &o, int K, std::vector<uint8_t> &blob,
                    ts_layout_info &info, std::string &err);

}  // namespace ts
