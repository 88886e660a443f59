// typerep.cpp -- layout-tree builders (see typerep.hpp).
//
// Each builder restates one helper of
// /root/reference/pkg/src/minimpi/datatype.py; line numbers are cited inline.
// The invariant they maintain (datatype.py:38-41): every node is non-empty
// except the Empty singleton, and traversal-adjacent runs are never
// byte-adjacent, so runs counts are maximal-segment counts.
#include "typerep.hpp"

#include <algorithm>
#include <stdexcept>

namespace mpx {
namespace tree {

namespace {
std::shared_ptr<Node> fresh(Kind k) {
    auto n = std::make_shared<Node>();
    n->kind = k;
    return n;
}
}  // namespace

const NodeP& empty() {
    static const NodeP e = fresh(Kind::Empty);
    return e;
}

NodeP run(int64_t off, int64_t len) {  // datatype.py:68-108
    auto n = fresh(Kind::Run);
    n->off = off;
    n->len = len;
    n->runs = 1;
    n->nbytes = len;
    n->first_start = n->min_off = off;
    n->last_end = n->max_end = off + len;
    return n;
}

NodeP rep(int64_t count, int64_t stride, NodeP body, int64_t base) {  // :124-137
    auto n = fresh(Kind::Rep);
    const Node& b = *body;
    const int64_t span = (count - 1) * stride;
    n->count = count;
    n->stride = stride;
    n->base = base;
    n->runs = count * b.runs;
    n->nbytes = count * b.nbytes;
    n->node_count = 1 + b.node_count;
    n->first_start = base + b.first_start;
    n->last_end = base + span + b.last_end;
    n->min_off = base + std::min<int64_t>(0, span) + b.min_off;
    n->max_end = base + std::max<int64_t>(0, span) + b.max_end;
    n->body = std::move(body);
    return n;
}

NodeP seq(std::vector<NodeP> kids) {  // :175-196
    auto n = fresh(Kind::Seq);
    const size_t k = kids.size();
    n->run_prefix.resize(k + 1);
    n->byte_prefix.resize(k + 1);
    n->run_prefix[0] = n->byte_prefix[0] = 0;
    int64_t nodes = 1, lo = kids[0]->min_off, hi = kids[0]->max_end;
    for (size_t i = 0; i < k; ++i) {
        const Node& c = *kids[i];
        n->run_prefix[i + 1] = n->run_prefix[i] + c.runs;
        n->byte_prefix[i + 1] = n->byte_prefix[i] + c.nbytes;
        nodes += c.node_count;
        lo = std::min(lo, c.min_off);
        hi = std::max(hi, c.max_end);
    }
    n->runs = n->run_prefix[k];
    n->nbytes = n->byte_prefix[k];
    n->node_count = nodes;
    n->first_start = kids.front()->first_start;
    n->last_end = kids.back()->last_end;
    n->min_off = lo;
    n->max_end = hi;
    n->kids = std::move(kids);
    return n;
}

NodeP shifted(const NodeP& n, int64_t d) {  // :218-225
    if (d == 0 || n->runs == 0) return n;
    switch (n->kind) {
    case Kind::Run: return run(n->off + d, n->len);
    case Kind::Rep: return rep(n->count, n->stride, n->body, n->base + d);
    default: {
        std::vector<NodeP> k;
        k.reserve(n->kids.size());
        for (const auto& c : n->kids) k.push_back(shifted(c, d));
        return seq(std::move(k));
    }
    }
}

void first_run(const Node* n, int64_t* off, int64_t* len) {  // :228-234
    int64_t acc = 0;
    while (n->kind != Kind::Run) {
        if (n->kind == Kind::Rep) { acc += n->base; n = n->body.get(); }
        else n = n->kids.front().get();
    }
    *off = acc + n->off;
    *len = n->len;
}

void last_run(const Node* n, int64_t* off, int64_t* len) {  // :237-243
    int64_t acc = 0;
    while (n->kind != Kind::Run) {
        if (n->kind == Kind::Rep) {
            acc += n->base + (n->count - 1) * n->stride;
            n = n->body.get();
        } else {
            n = n->kids.back().get();
        }
    }
    *off = acc + n->off;
    *len = n->len;
}

NodeP seq_raw(const std::vector<NodeP>& parts) {  // :246-259
    std::vector<NodeP> flat;
    const NodeP* only = nullptr;
    size_t kept = 0;
    for (const auto& p : parts) {
        if (p->runs == 0) continue;
        ++kept;
        only = &p;
        if (p->kind == Kind::Seq) flat.insert(flat.end(), p->kids.begin(), p->kids.end());
        else flat.push_back(p);
    }
    if (kept == 0) return empty();
    if (kept == 1) return *only;
    return seq(std::move(flat));
}

NodeP make_rep(int64_t count, int64_t stride, const NodeP& body, int64_t base) {  // :262-267
    if (count <= 0 || body->runs == 0) return empty();
    if (count == 1) return shifted(body, base);
    return rep(count, stride, body, base);
}

NodeP drop_first(const NodeP& n) {  // :270-280
    switch (n->kind) {
    case Kind::Run: return empty();
    case Kind::Rep: {
        NodeP rest = make_rep(n->count - 1, n->stride, n->body, n->base + n->stride);
        if (n->body->runs == 1) return rest;
        return seq_raw({shifted(drop_first(n->body), n->base), rest});
    }
    default: {
        std::vector<NodeP> p(n->kids);
        p.front() = drop_first(p.front());
        return seq_raw(p);
    }
    }
}

NodeP drop_last(const NodeP& n) {  // :283-293
    switch (n->kind) {
    case Kind::Run: return empty();
    case Kind::Rep: {
        NodeP head = make_rep(n->count - 1, n->stride, n->body, n->base);
        if (n->body->runs == 1) return head;
        const int64_t last_base = n->base + (n->count - 1) * n->stride;
        return seq_raw({head, shifted(drop_last(n->body), last_base)});
    }
    default: {
        std::vector<NodeP> p(n->kids);
        p.back() = drop_last(p.back());
        return seq_raw(p);
    }
    }
}

NodeP replicate(const NodeP& body, int64_t count, int64_t stride) {  // :296-315
    if (body->runs == 0 || count == 0) return empty();
    if (count == 1) return body;
    if (body->last_end != stride + body->first_start) return rep(count, stride, body, 0);
    // the last run of each copy is flush against the first run of the next
    if (body->runs == 1) return run(body->first_start, (count - 1) * stride + body->nbytes);
    int64_t h_off, h_len, t_off, t_len;
    first_run(body.get(), &h_off, &h_len);
    last_run(body.get(), &t_off, &t_len);
    NodeP mid = drop_last(drop_first(body));
    NodeP inner = seq_raw({mid, run(t_off, t_len + h_len)});
    NodeP tail = shifted(drop_first(body), (count - 1) * stride);
    return seq_raw({run(h_off, h_len), make_rep(count - 1, stride, inner, 0), tail});
}

NodeP concat(const std::vector<NodeP>& parts) {  // :318-337
    std::vector<NodeP> acc;
    acc.reserve(parts.size());
    for (const auto& p : parts) {
        if (p->runs == 0) continue;
        if (!acc.empty() && acc.back()->last_end == p->first_start) {
            NodeP prev = acc.back();
            acc.pop_back();
            int64_t t_off, t_len, h_off, h_len;
            last_run(prev.get(), &t_off, &t_len);
            first_run(p.get(), &h_off, &h_len);
            NodeP rem = drop_last(prev);
            if (rem->runs) acc.push_back(rem);
            acc.push_back(run(t_off, t_len + h_len));
            NodeP rest = drop_first(p);
            if (rest->runs) acc.push_back(rest);
        } else {
            acc.push_back(p);
        }
    }
    return seq_raw(acc);
}

void prefix_within(const Node* n, int64_t budget, int64_t* segs, int64_t* used) {
    // RUN :105-108, REP :155-163, SEQ :208-215 -- iterative descent
    *segs = 0;
    *used = 0;
    for (;;) {
        switch (n->kind) {
        case Kind::Empty: return;
        case Kind::Run:
            if (n->len <= budget) { *segs += 1; *used += n->len; }
            return;
        case Kind::Rep: {
            const int64_t per = n->body->nbytes;
            const int64_t q = std::min(budget / per, n->count);
            *segs += q * n->body->runs;
            *used += q * per;
            if (q >= n->count) return;
            budget -= q * per;
            n = n->body.get();
            break;
        }
        case Kind::Seq: {
            const auto& bp = n->byte_prefix;
            const size_t i = size_t(std::upper_bound(bp.begin(), bp.end(), budget) - bp.begin()) - 1;
            *segs += n->run_prefix[i];
            *used += bp[i];
            if (i >= n->kids.size()) return;
            budget -= bp[i];
            n = n->kids[i].get();
            break;
        }
        }
    }
}

void enumerate(const Node* n, int64_t shift, std::vector<int64_t>& out, int64_t limit) {
    if ((int64_t)out.size() >= 2 * limit) return;
    switch (n->kind) {
    case Kind::Empty: return;
    case Kind::Run:
        out.push_back(shift + n->off);
        out.push_back(n->len);
        return;
    case Kind::Rep:
        for (int64_t k = 0; k < n->count && (int64_t)out.size() < 2 * limit; ++k)
            enumerate(n->body.get(), shift + n->base + k * n->stride, out, limit);
        return;
    case Kind::Seq:
        for (const auto& c : n->kids) enumerate(c.get(), shift, out, limit);
        return;
    }
}

int depth(const Node* n) {
    switch (n->kind) {
    case Kind::Empty:
    case Kind::Run: return 1;
    case Kind::Rep: return 1 + depth(n->body.get());
    default: {
        int d = 0;
        for (const auto& c : n->kids) d = std::max(d, depth(c.get()));
        return 1 + d;
    }
    }
}

}  // namespace tree

NodeP Datatype::layout_for(int64_t count) {  // datatype.py:658-661
    if (count == 1) return layout;
    std::lock_guard<std::mutex> g(mu);
    auto it = replicated.find(count);
    if (it != replicated.end()) return it->second;
    NodeP l = tree::replicate(layout, count, extent());
    if (replicated.size() > 64) replicated.clear();
    replicated.emplace(count, l);
    return l;
}

}  // namespace mpx
