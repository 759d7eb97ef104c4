// ref_sbp_rule — the UNMODIFIED reference's SBP rule loader (quadrature.hpp:290-343) on
// a caller's file, printed as hex floats — TEST INFRASTRUCTURE (built into oracle/_ref/
// by oracle/Makefile.ref; tests/test_sbp_rule_file.py compares the native setup's
// loader with it).
//
//   ref_sbp_rule N family(0 legendre | 1 lobatto) data_dir|- rule_file|-
// prints "ok nq npf", then nq lines "x y w" (%a), then the face_node_index line;
// or "error <message>" (exit 1).
#include <cstdio>
#include <string>

#include "swedg/quadrature.hpp"

using namespace swedg;

int main(int argc, char** argv) {
    if (argc < 5) return 2;
    const int N = std::atoi(argv[1]);
    const EdgeFamily fam = std::atoi(argv[2]) ? EdgeFamily::GaussLobatto : EdgeFamily::GaussLegendre;
    const std::string dir = argv[3], file = argv[4];
    try {
        SBPQuadrature q = file != "-" ? load_sbp_rule_file(file, N, fam) : sbp_rule(N, fam, dir == "-" ? "" : dir);
        std::printf("ok %d %d\n", q.vol.size(), q.surf.nodes_per_face);
        for (int i = 0; i < q.vol.size(); ++i) std::printf("%a %a %a\n", q.vol.x[i], q.vol.y[i], q.vol.w[i]);
        for (int v : q.face_node_index) std::printf("%d ", v);
        std::printf("\n");
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
    return 0;
}
