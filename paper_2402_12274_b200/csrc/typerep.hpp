// typerep.hpp -- host-side derived-datatype compiler.
//
// Builds the reference's constant-size layout tree
// (/root/reference/pkg/src/minimpi/datatype.py:45-337): Run / Rep / Seq nodes
// with cached segment counts and byte totals, assembled by merge-resolving
// builders so that node->runs is exactly the maximal contiguous-run count the
// reference reports.  Trees are immutable DAGs shared between datatypes
// (std::shared_ptr<const Node>).  The tree is then lowered to a GPU plan
// (plan.hpp): a closed-form strided chain when the tree is Rep^k(Run), or a
// flat device descriptor walked by the generic kernels otherwise.
#pragma once

#include <cstdint>
#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace mpx {

enum class Kind : int32_t { Empty = 0, Run = 1, Rep = 2, Seq = 3 };

struct Node;
using NodeP = std::shared_ptr<const Node>;

struct Node {
    Kind kind = Kind::Empty;
    // Run
    int64_t off = 0, len = 0;
    // Rep: count copies of body, copy k displaced by base + k*stride
    int64_t count = 0, stride = 0, base = 0;
    NodeP body;
    // Seq: heterogeneous children, offsets pre-shifted
    std::vector<NodeP> kids;
    std::vector<int64_t> run_prefix, byte_prefix;
    // cached summary (datatype.py:118-137, 175-196)
    int64_t runs = 0, nbytes = 0, node_count = 1;
    int64_t first_start = 0, last_end = 0, min_off = 0, max_end = 0;
};

namespace tree {
const NodeP& empty();
NodeP run(int64_t off, int64_t len);
NodeP rep(int64_t count, int64_t stride, NodeP body, int64_t base);
NodeP seq(std::vector<NodeP> kids);
NodeP shifted(const NodeP& n, int64_t d);
void first_run(const Node* n, int64_t* off, int64_t* len);
void last_run(const Node* n, int64_t* off, int64_t* len);
NodeP seq_raw(const std::vector<NodeP>& parts);
NodeP make_rep(int64_t count, int64_t stride, const NodeP& body, int64_t base);
NodeP drop_first(const NodeP& n);
NodeP drop_last(const NodeP& n);
NodeP replicate(const NodeP& body, int64_t count, int64_t stride);
NodeP concat(const std::vector<NodeP>& parts);
// (segments, bytes) of whole leading segments within budget
void prefix_within(const Node* n, int64_t budget, int64_t* segs, int64_t* used);
// host enumeration used only for plan analysis (overlap test) on small trees
void enumerate(const Node* n, int64_t shift, std::vector<int64_t>& out, int64_t limit);
int depth(const Node* n);
}  // namespace tree

struct Plan;  // plan.hpp

// A committed or uncommitted datatype (datatype.py:345-407).
struct Datatype {
    NodeP layout;
    int64_t size = 0, lb = 0, ub = 0;
    bool committed = false, freed = false, builtin = false;
    std::string desc;

    int64_t extent() const { return ub - lb; }

    // per-(device, count) lowered plans, built lazily on first data movement
    std::mutex mu;
    std::map<std::pair<int, int64_t>, std::shared_ptr<Plan>> plans;
    std::map<int64_t, NodeP> replicated;  // layout_for(count) cache
    std::map<int64_t, std::array<int64_t, 8>> queries;   // mpx_layout_query(count) cache

    NodeP layout_for(int64_t count);      // datatype.py:658-661
};

}  // namespace mpx
