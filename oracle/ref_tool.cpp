// oracle/ref_tool.cpp -- the reference's stream-based writers as a command
// (test infrastructure): write_pfm / write_text_matrix, hash_file,
// stats_lines.  Compiled against the unmodified reference headers.
#include <tofr/pipeline.hpp>

#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

using namespace tofr;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::string verb = argv[1];
    if (verb == "write_image" && argc == 7) {  // raw.f64 w h out.pfm out.txt
        int w = std::atoi(argv[3]), h = std::atoi(argv[4]);
        std::vector<double> buf(size_t(w) * h * 3);
        FILE* f = std::fopen(argv[2], "rb");
        if (!f || std::fread(buf.data(), 8, buf.size(), f) != buf.size()) return 2;
        std::fclose(f);
        Image img(w, h);
        for (size_t i = 0; i < size_t(w) * h; ++i) img.px[i] = {buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]};
        write_pfm(img, argv[5]);
        write_text_matrix(img, argv[6]);
        return 0;
    }
    if (verb == "hash" && argc == 3) {
        std::cout << hash_file(argv[2]) << "\n";
        return 0;
    }
    if (verb == "stats_lines") {  // stdin: frame t_init t_shade then 3 x (9 counters, seconds)
        std::vector<FrameStats> stats;
        std::string line;
        while (std::getline(std::cin, line)) {
            if (line.empty()) continue;
            std::istringstream ls(line);
            FrameStats fs;
            ls >> fs.frame >> fs.t_init >> fs.t_shade;
            for (StageStats* st : {&fs.temporal, &fs.spatial, &fs.binwise}) {
                ShiftCounts& c = st->shift;
                ls >> c.attempts >> c.newton_ok >> c.newton_failed >> c.occluded >> c.jac_clamped >>
                    c.replay_failed >> c.iterations >> c.solves >> c.success >> st->seconds;
            }
            stats.push_back(fs);
        }
        std::cout << stats_lines(stats);
        return 0;
    }
    return 2;
}
