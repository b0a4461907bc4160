// mvm_b200.cpp -- link-substitutes for the reference's compressed MVMs (the finer-grained
// drop-ins of SURVEY.md section 8b):
//   dax_mvm  (dax.hpp:37, dax.cpp:96-103)  -> qcs_dax_mvm
//   das_mvm  (das.hpp:39, das.cpp:131-150) -> qcs_das_mvm
//   rh_mvm   (rh.hpp:64-66, rh.cpp:92-156) -> qcs_rh_mvm (RhMvmStats filled as the reference does)
// Each keeps the reference's signature, value semantics, checks and messages; the operator and
// the state go to the device, the product comes back as a fresh StateVector.
// The reference defines these next to functions the shim does not replace (dax_encode, dax_mtp,
// the dumps ...), so oracle/Makefile links the reference's own dax.o / das.o / rh.o with the three
// symbols weakened (objcopy --weaken-symbol); INTEGRATION.md shows the same swap for a CMake build.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "qcsim/dax.hpp"
#include "qcsim/das.hpp"
#include "qcsim/rh.hpp"
#include "shim_common.hpp"

namespace qcsim {

using b200::check;

namespace {

// upload s into the pool's input slot, run `op(in, out)`, download the output slot
template <class Op>
StateVector run_mvm(const StateVector& s, Op op) {
    StateVector out;
    out.n = s.n;
    out.amps.assign(s.dim(), cplx{0.0, 0.0});
    if (s.dim() == 0) return out;
    const int q = b200::qubits_of(s.dim());
    qcs_state* in = b200::pool().get(b200::kMvmIn, q);
    qcs_state* o = b200::pool().get(b200::kMvmOut, q);
    check(qcs_state_upload(in, reinterpret_cast<const double*>(s.amps.data()), 0, s.dim()));
    op(in, o);
    check(qcs_state_download(o, reinterpret_cast<double*>(out.amps.data()), 0, s.dim()));
    return out;
}

}  // namespace

StateVector dax_mvm(const DaxMatrix& m, const StateVector& s) {
    if (m.rows != m.cols || m.cols != s.dim()) throw DimensionError("DAX MVM shape mismatch");
    const std::size_t cnt = m.entries.size();
    // the device kernel finds a row's entries by binary search, so it takes them grouped by
    // row; a stable order by row keeps each row's accumulation order, i.e. the reference's
    // result bit for bit even for a DaxMatrix that breaks its sortedness invariant (dax.hpp:20)
    std::vector<std::size_t> order;
    bool sorted = true;
    for (std::size_t i = 1; i < cnt && sorted; ++i) sorted = m.entries[i - 1].row <= m.entries[i].row;
    if (!sorted) {
        order.resize(cnt);
        std::iota(order.begin(), order.end(), std::size_t(0));
        std::stable_sort(order.begin(), order.end(),
                         [&](std::size_t a, std::size_t b) { return m.entries[a].row < m.entries[b].row; });
    }
    std::vector<std::uint64_t> rows(cnt), cols(cnt);
    std::vector<cplx> vals(cnt);
    for (std::size_t i = 0; i < cnt; ++i) {
        const DaxEntry& e = m.entries[sorted ? i : order[i]];
        if (e.row >= m.rows || e.col >= m.cols) throw DimensionError("DAX MVM entry out of range");
        rows[i] = e.row;
        cols[i] = e.col;
        vals[i] = e.value;
    }
    return run_mvm(s, [&](qcs_state* in, qcs_state* out) {
        check(qcs_dax_mvm(rows.data(), cols.data(), reinterpret_cast<const double*>(vals.data()), cnt,
                          QCS_MEM_HOST, in, out));
    });
}

StateVector das_mvm(const DasMatrix& m, const StateVector& s) {
    if (m.rows != m.cols || m.cols != s.dim()) throw DimensionError("DAS MVM shape mismatch");
    const std::size_t cnt = m.entries.size();
    std::vector<std::uint64_t> dis(cnt);
    std::vector<std::uint8_t> last(cnt);
    std::vector<cplx> vals(cnt);
    for (std::size_t i = 0; i < cnt; ++i) {
        dis[i] = m.entries[i].dis;
        last[i] = m.entries[i].last_in_row ? 1 : 0;
        vals[i] = m.entries[i].value;
    }
    return run_mvm(s, [&](qcs_state* in, qcs_state* out) {
        check(qcs_das_mvm(dis.data(), last.data(), reinterpret_cast<const double*>(vals.data()), cnt, QCS_MEM_HOST,
                          in, out));  // malformed streams: EncodingError "malformed DAS stream" (das.cpp:140)
    });
}

StateVector rh_mvm(const RhMatrix& m, const StateVector& s, SignMethod method, RhMvmStats* stats,
                   std::uint64_t block_size) {
    if (m.n < 1) throw DimensionError("RH MVM needs n >= 1");
    if (s.n != m.n) throw DimensionError("RH MVM qubit count mismatch");
    std::uint64_t signs = 0, madds = 0;
    StateVector out = s;
    const int q = b200::qubits_of(s.dim());
    qcs_state* st = b200::pool().get(b200::kMvmIn, q);
    check(qcs_state_upload(st, reinterpret_cast<const double*>(s.amps.data()), 0, s.dim()));
    check(qcs_rh_mvm(st, m.n, m.value, int(method), block_size, &signs, &madds));
    check(qcs_state_download(st, reinterpret_cast<double*>(out.amps.data()), 0, s.dim()));
    if (stats) {
        stats->sign_count = signs;
        stats->madd_count = madds;
    }
    return out;
}

}  // namespace qcsim
