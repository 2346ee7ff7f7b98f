// The reference's wire-format writers/readers as a command-line tool (test
// infrastructure; the iostreams of the statically linked runtime cannot be
// used from inside the dlopen'ed libpstokes_ref.so):
//   wire_ref mesh <kind 0 family|1 quad|2 tri> <family> <n> <jitter> <side> <out>
//       write_mesh (mesh.hpp:540-560) of the mesh ref_system_create builds
//   wire_ref mtx <kind> <family> <n> <jitter> <side> <scheme> <strategy> <k> <out>
//       write_matrix_market (csr.hpp:98-111) of the assembled operator
//   wire_ref roundtrip <in> <out>
//       read_mesh (mesh.hpp:562-645) then write_mesh; prints "nv ne nf"
// Errors: the exception message on stderr, exit code 1.
#include "ref_driver.cpp"

#include <cstdio>
#include <cstdlib>

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "roundtrip" && argc == 4) {
      const Mesh m = read_mesh(std::string(argv[2]));
      write_mesh(m, std::string(argv[3]));
      std::printf("%d %d %d\n", m.n_vertices(), m.n_elements(), m.n_faces());
      return 0;
    }
    if ((cmd == "mesh" && argc == 8) || (cmd == "mtx" && argc == 11)) {
      const int kind = std::atoi(argv[2]);
      const int n = std::atoi(argv[4]);
      const double jit = std::atof(argv[5]);
      const Side side = static_cast<Side>(std::atoi(argv[6]));
      const Mesh m = kind == 0 ? make_family_mesh(argv[3], n, 1, side)
                               : unit_square_mesh(n, kind == 2, jit, 0, side);
      if (cmd == "mesh") {
        write_mesh(m, std::string(argv[7]));
        return 0;
      }
      const StokesSystem s = assemble_stokes(m, static_cast<Scheme>(std::atoi(argv[7])),
                                             static_cast<Strategy>(std::atoi(argv[8])),
                                             std::atoi(argv[9]), ManufacturedCase::data(), 0.0);
      write_matrix_market(s.a, std::string(argv[10]));
      return 0;
    }
    std::fprintf(stderr, "usage: see oracle/wire_ref.cpp\n");
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
}
