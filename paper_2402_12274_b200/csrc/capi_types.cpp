// capi_types.cpp -- extern "C" datatype / pack / unpack / iov entry points.
//
// Argument validation mirrors the reference (datatype.py:403-436, 618-692)
// and happens on the host at call time; the data movement itself is enqueued
// asynchronously on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>

#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_set>
#include <vector>

#include "capi_common.hpp"
#include "kernels.hpp"
#include "mpx.h"
#include "plan.hpp"
#include "typerep.hpp"

using namespace mpx;

namespace mpx {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(MPX_ERR_OTHER, "%s: %s", what, cudaGetErrorString(e));
}

namespace {
std::mutex g_reg_mu;
std::unordered_set<const void*> g_registry;

Datatype* make_builtin(int64_t size, const char* name) {
    auto* d = new Datatype();
    d->layout = tree::run(0, size);
    d->size = size;
    d->lb = 0;
    d->ub = size;
    d->committed = true;
    d->builtin = true;
    d->desc = name;
    std::lock_guard<std::mutex> g(g_reg_mu);
    g_registry.insert(d);
    return d;
}

Datatype* builtin(int which) {
    static Datatype* table[7] = {
        make_builtin(1, "byte"),   make_builtin(1, "char"),    make_builtin(1, "int8"),
        make_builtin(4, "int32"),  make_builtin(8, "int64"),   make_builtin(4, "float32"),
        make_builtin(8, "float64")};
    if (which < 0 || which > 6) return nullptr;
    return table[which];
}

mpx_datatype publish(Datatype* d) {
    std::lock_guard<std::mutex> g(g_reg_mu);
    g_registry.insert(d);
    return reinterpret_cast<mpx_datatype>(d);
}
}  // namespace

Datatype* lookup(mpx_datatype h) {
    std::lock_guard<std::mutex> g(g_reg_mu);
    auto* d = reinterpret_cast<Datatype*>(h);
    return g_registry.count(d) ? d : nullptr;
}

namespace {
// _check_child: datatype.py:425-431
int check_child(mpx_datatype h, Datatype** out) {
    Datatype* d = lookup(h);
    if (!d) return fail(MPX_ERR_ARG, "child must be a Datatype");
    if (d->freed) return fail(MPX_ERR_ARG, "child datatype was freed");
    if (!d->committed) return fail(MPX_ERR_ARG, "child datatype must be committed (or basic)");
    *out = d;
    return MPX_SUCCESS;
}

int check_count(int64_t n, const char* what) {  // datatype.py:434-436
    if (n < 0) return fail(MPX_ERR_ARG, "%s must be an integer >= 0", what);
    return MPX_SUCCESS;
}

// _check_usable: datatype.py:403-407
int check_usable(Datatype* d, const char* what) {
    if (!d) return fail(MPX_ERR_ARG, "not a datatype handle");
    if (d->freed) return fail(MPX_ERR_ARG, "datatype %s after free", what);
    if (!d->committed) return fail(MPX_ERR_ARG, "datatype %s before commit", what);
    return MPX_SUCCESS;
}

Datatype* new_type(NodeP lay, int64_t size, int64_t lb, int64_t ub, std::string desc) {
    auto* d = new Datatype();
    d->layout = std::move(lay);
    d->size = size;
    d->lb = lb;
    d->ub = ub;
    d->desc = std::move(desc);
    return d;
}

// Where a buffer lives.  Device memory -> its device.  Pinned / registered
// host memory is accepted too (*dev = -1): kernels address it directly over
// PCIe through its UVA device pointer (zero-copy).  Pageable memory is refused.
int resolve_ptr(const void* p, int* dev) {
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(MPX_ERR_ARG, "cannot resolve buffer %p: %s", p, cudaGetErrorString(e));
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        *dev = a.device;
        return MPX_SUCCESS;
    }
    if (a.type == cudaMemoryTypeHost) {
        if (a.devicePointer != p)
            return fail(MPX_ERR_ARG, "pinned host buffer %p is not mapped at the same UVA address", p);
        *dev = -1;
        return MPX_SUCCESS;
    }
    return fail(MPX_ERR_ARG, "buffer %p is pageable host memory: pass a CUDA tensor or pinned memory", p);
}

int device_of(const void* p, int* dev) {
    int rc = resolve_ptr(p, dev);
    if (rc == MPX_SUCCESS && *dev < 0) cudaGetDevice(dev);
    return rc;
}

// execution device for an operation touching buffers a and b
int device_for(const void* a, const void* b, int* dev) {
    int da = -1, db = -1, rc;
    if ((rc = resolve_ptr(a, &da)) || (rc = resolve_ptr(b, &db))) return rc;
    if (da >= 0 && db >= 0 && da != db)
        return fail(MPX_ERR_ARG, "buffers live on different devices (%d, %d)", da, db);
    *dev = da >= 0 ? da : db;
    if (*dev < 0) cudaGetDevice(dev);
    return MPX_SUCCESS;
}

int ensure_device(int dev) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != dev) {
        cudaError_t e = cudaSetDevice(dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    }
    return MPX_SUCCESS;
}
}  // namespace

// Validate + lower one pack/unpack operation.  layout_buf is the typed side.
int prepare(Datatype* d, int64_t count, const void* layout_buf, int64_t layout_bytes, const void* other_buf,
            cudaStream_t stream, std::shared_ptr<Plan>* plan, int* device) {
    int rc = check_count(count, "count");
    if (rc) return rc;
    rc = check_usable(d, "pack/unpack");
    if (rc) return rc;
    NodeP lay = d->layout_for(count);
    if (lay->runs) {  // _checked_view bounds, datatype.py:685-691
        if (lay->min_off < 0) return fail(MPX_ERR_ARG, "layout reaches before the start of the buffer");
        if (lay->max_end > layout_bytes)
            return fail(MPX_ERR_ARG, "buffer too small: layout spans %lld bytes, buffer has %lld",
                        (long long)lay->max_end, (long long)layout_bytes);
    }
    if (lay->runs == 0) {
        *plan = nullptr;
        return MPX_SUCCESS;
    }
    int dev = 0;
    rc = device_for(layout_buf, other_buf ? other_buf : layout_buf, &dev);
    if (rc) return rc;
    rc = ensure_device(dev);
    if (rc) return rc;
    std::string err;
    *plan = get_plan(d, count, dev, stream, &err);
    if (!*plan) return fail(MPX_ERR_OTHER, "%s", err.c_str());
    *device = dev;
    return MPX_SUCCESS;
}

}  // namespace mpx

extern "C" {

int mpx_abi_version(void) { return 1; }

const char* mpx_last_error(void) { return g_last_error.c_str(); }

int mpx_device_set_l2_fetch(int device, int bytes, int* prev) {
    int rc = ensure_device(device);
    if (rc) return rc;
    size_t old = 0;
    cudaError_t e = cudaDeviceGetLimit(&old, cudaLimitMaxL2FetchGranularity);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetLimit");
    if (prev) *prev = (int)old;
    if (bytes >= 0) {
        e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSetLimit(L2 fetch)");
    }
    return MPX_SUCCESS;
}

int mpx_type_builtin(int which, mpx_datatype* out) {
    Datatype* d = builtin(which);
    if (!d || !out) return fail(MPX_ERR_ARG, "unknown builtin %d", which);
    *out = reinterpret_cast<mpx_datatype>(d);
    return MPX_SUCCESS;
}

int mpx_type_contiguous(int64_t count, mpx_datatype child, mpx_datatype* out) {
    Datatype* c = nullptr;
    int rc = check_count(count, "count");
    if (rc || (rc = check_child(child, &c))) return rc;
    const int64_t ext = c->extent();
    NodeP lay = tree::replicate(c->layout, count, ext);
    int64_t lb = 0, ub = 0;
    if (count) { lb = c->lb; ub = (count - 1) * ext + c->ub; }
    *out = publish(new_type(lay, count * c->size, lb, ub,
                            "contiguous(" + std::to_string(count) + ", " + c->desc + ")"));
    return MPX_SUCCESS;
}

static int vector_like(int64_t count, int64_t bl, int64_t step, mpx_datatype child, mpx_datatype* out,
                       const std::string& what) {
    Datatype* c = nullptr;
    int rc = check_count(count, "count");
    if (rc || (rc = check_count(bl, "blocklength")) || (rc = check_child(child, &c))) return rc;
    const int64_t ext = c->extent();
    NodeP block = tree::replicate(c->layout, bl, ext);
    NodeP lay = tree::replicate(block, count, step);
    int64_t lb = 0, ub = 0;
    if (count && bl) {
        const int64_t span = (count - 1) * step;
        lb = std::min<int64_t>(0, span) + c->lb;
        ub = std::max<int64_t>(0, span) + (bl - 1) * ext + c->ub;
    }
    *out = publish(new_type(lay, count * bl * c->size, lb, ub, what + ", " + c->desc + ")"));
    return MPX_SUCCESS;
}

int mpx_type_vector(int64_t count, int64_t bl, int64_t stride, mpx_datatype child, mpx_datatype* out) {
    Datatype* c = lookup(child);
    const int64_t ext = c ? c->extent() : 0;
    return vector_like(count, bl, stride * ext, child, out,
                       "vector(" + std::to_string(count) + ", " + std::to_string(bl) + ", " +
                           std::to_string(stride));
}

int mpx_type_hvector(int64_t count, int64_t bl, int64_t stride_bytes, mpx_datatype child,
                     mpx_datatype* out) {
    return vector_like(count, bl, stride_bytes, child, out,
                       "hvector(" + std::to_string(count) + ", " + std::to_string(bl) + ", " +
                           std::to_string(stride_bytes) + "b");
}

int mpx_type_indexed_block(int64_t bl, int64_t n, const int64_t* displs, mpx_datatype child,
                           mpx_datatype* out) {
    Datatype* c = nullptr;
    int rc = check_count(bl, "blocklength");
    if (rc || (rc = check_child(child, &c))) return rc;
    if (n < 0 || (n && !displs)) return fail(MPX_ERR_ARG, "displacements must be integers");
    const int64_t ext = c->extent();
    NodeP block = tree::replicate(c->layout, bl, ext);
    std::vector<NodeP> parts;
    parts.reserve(n);
    int64_t dmin = 0, dmax = 0;
    for (int64_t i = 0; i < n; ++i) {
        parts.push_back(tree::shifted(block, displs[i] * ext));
        dmin = i ? std::min(dmin, displs[i]) : displs[i];
        dmax = i ? std::max(dmax, displs[i]) : displs[i];
    }
    int64_t lb = 0, ub = 0;
    if (n && bl) { lb = dmin * ext + c->lb; ub = (dmax + bl - 1) * ext + c->ub; }
    *out = publish(new_type(tree::concat(parts), n * bl * c->size, lb, ub,
                            "indexed_block(" + std::to_string(bl) + ", n=" + std::to_string(n) + ", " +
                                c->desc + ")"));
    return MPX_SUCCESS;
}

static int struct_like(int64_t n, const int64_t* bls, const int64_t* displs, Datatype* const* kids,
                       bool scale_by_extent, mpx_datatype* out, const std::string& desc) {
    std::vector<NodeP> parts;
    parts.reserve(n);
    int64_t size = 0, lb = 0, ub = 0;
    bool have = false;
    for (int64_t i = 0; i < n; ++i) {
        int rc = check_count(bls[i], "blocklength");
        if (rc) return rc;
        Datatype* c = kids[i];
        const int64_t ext = c->extent();
        const int64_t d = scale_by_extent ? displs[i] * ext : displs[i];
        parts.push_back(tree::shifted(tree::replicate(c->layout, bls[i], ext), d));
        size += bls[i] * c->size;
        if (bls[i] > 0) {
            const int64_t b_lb = d + c->lb, b_ub = d + (bls[i] - 1) * ext + c->ub;
            lb = have ? std::min(lb, b_lb) : b_lb;
            ub = have ? std::max(ub, b_ub) : b_ub;
            have = true;
        }
    }
    *out = publish(new_type(tree::concat(parts), size, lb, ub, desc));
    return MPX_SUCCESS;
}

int mpx_type_indexed(int64_t n, const int64_t* bls, const int64_t* displs, mpx_datatype child,
                     mpx_datatype* out) {
    Datatype* c = nullptr;
    int rc = check_child(child, &c);
    if (rc) return rc;
    if (n < 0 || (n && (!bls || !displs))) return fail(MPX_ERR_ARG, "indexed arrays must have equal length");
    std::vector<Datatype*> kids(n, c);
    return struct_like(n, bls, displs, kids.data(), true, out,
                       "indexed(n=" + std::to_string(n) + ", " + c->desc + ")");
}

int mpx_type_create_struct(int64_t n, const int64_t* bls, const int64_t* displs,
                           const mpx_datatype* children, mpx_datatype* out) {
    if (n < 0 || (n && (!bls || !displs || !children)))
        return fail(MPX_ERR_ARG, "struct arrays must have equal length");
    std::vector<Datatype*> kids(n);
    std::string desc = "struct(";
    for (int64_t i = 0; i < n; ++i) {
        int rc = check_child(children[i], &kids[i]);
        if (rc) return rc;
        desc += (i ? ", " : "") + std::to_string(bls[i]) + "x" + kids[i]->desc + "@" + std::to_string(displs[i]);
    }
    return struct_like(n, bls, displs, kids.data(), false, out, desc + ")");
}

int mpx_type_create_subarray(int nd, const int64_t* full, const int64_t* sub, const int64_t* offs,
                             mpx_datatype child, mpx_datatype* out) {
    if (nd < 1 || !full || !sub || !offs)
        return fail(MPX_ERR_ARG, "subarray dimension arrays must match and be non-empty");
    for (int i = 0; i < nd; ++i) {
        int rc;
        if ((rc = check_count(full[i], "full size")) || (rc = check_count(sub[i], "sub size")) ||
            (rc = check_count(offs[i], "offset")))
            return rc;
        if (sub[i] > full[i] || offs[i] > full[i] - sub[i])
            return fail(MPX_ERR_ARG, "subarray block must fit inside the full array");
    }
    Datatype* c = nullptr;
    int rc = check_child(child, &c);
    if (rc) return rc;
    const int64_t ext = c->extent();
    std::vector<int64_t> st(nd);
    st[nd - 1] = ext;
    for (int k = nd - 2; k >= 0; --k) st[k] = st[k + 1] * full[k + 1];
    NodeP core = tree::replicate(c->layout, sub[nd - 1], ext);
    for (int k = nd - 2; k >= 0; --k) core = tree::replicate(core, sub[k], st[k]);
    int64_t base = 0, size = c->size, vol = 1;
    for (int k = 0; k < nd; ++k) {
        base += offs[k] * st[k];
        size *= sub[k];
        vol *= full[k];
    }
    *out = publish(new_type(tree::shifted(core, base), size, 0, vol * ext,
                            "subarray(nd=" + std::to_string(nd) + ", " + c->desc + ")"));
    return MPX_SUCCESS;
}

int mpx_type_create_resized(mpx_datatype child, int64_t lb, int64_t extent, mpx_datatype* out) {
    Datatype* c = nullptr;
    int rc = check_child(child, &c);
    if (rc) return rc;
    if (extent < 0) return fail(MPX_ERR_ARG, "resized needs integer lb and extent >= 0");
    *out = publish(new_type(c->layout, c->size, lb, lb + extent,
                            "resized(" + c->desc + ", lb=" + std::to_string(lb) + ", extent=" +
                                std::to_string(extent) + ")"));
    return MPX_SUCCESS;
}

int mpx_type_commit(mpx_datatype h) {  // datatype.py:594-600
    Datatype* d = lookup(h);
    if (!d) return fail(MPX_ERR_ARG, "type_commit expects a Datatype");
    if (d->freed) return fail(MPX_ERR_ARG, "cannot commit a freed datatype");
    d->committed = true;
    return MPX_SUCCESS;
}

int mpx_type_free(mpx_datatype h) {  // datatype.py:603-610
    Datatype* d = lookup(h);
    if (!d) return fail(MPX_ERR_ARG, "type_free expects a Datatype");
    if (d->builtin) return fail(MPX_ERR_ARG, "builtin datatypes cannot be freed");
    if (d->freed) return fail(MPX_ERR_ARG, "datatype already freed");
    d->freed = true;
    std::lock_guard<std::mutex> g(d->mu);
    d->plans.clear();       // releases device descriptors
    d->replicated.clear();
    return MPX_SUCCESS;
}

int mpx_type_get_info(mpx_datatype h, int64_t info[8]) {
    Datatype* d = lookup(h);
    if (!d) return fail(MPX_ERR_ARG, "not a datatype handle");
    info[0] = d->size;
    info[1] = d->lb;
    info[2] = d->ub;
    info[3] = d->extent();
    info[4] = d->layout->runs;
    info[5] = d->layout->node_count;
    info[6] = d->committed;
    info[7] = d->freed;
    return MPX_SUCCESS;
}

int mpx_type_iov_len(mpx_datatype h, int64_t max_bytes, int64_t* n, int64_t* bytes) {
    Datatype* d = lookup(h);
    int rc = check_usable(d, "query");
    if (rc) return rc;
    if (max_bytes < -1) return fail(MPX_ERR_ARG, "max_iov_bytes must be an integer >= -1");
    if (max_bytes == -1 || max_bytes >= d->size) {
        *n = d->layout->runs;
        *bytes = d->size;
        return MPX_SUCCESS;
    }
    tree::prefix_within(d->layout.get(), max_bytes, n, bytes);
    return MPX_SUCCESS;
}

int mpx_packed_size(mpx_datatype h, int64_t count, int64_t* out) {
    Datatype* d = lookup(h);
    int rc = check_count(count, "count");
    if (rc || (rc = check_usable(d, "size query"))) return rc;
    *out = d->size * count;
    return MPX_SUCCESS;
}

int mpx_plan_dump(mpx_datatype h, int64_t count, int64_t* out, int64_t cap, int64_t* n) {
    Datatype* d = lookup(h);
    int rc = check_count(count, "count");
    if (rc || (rc = check_usable(d, "query"))) return rc;
    NodeP lay = d->layout_for(count);
    Plan p;
    analyze(lay.get(), &p);
    std::vector<int64_t> v;
    v.push_back(p.kind);
    v.push_back(p.span.outer_depth);
    for (int i = 0; i < kSpanMaxOuter; ++i) {
        v.push_back(p.span.outer_cnt[i]);
        v.push_back(p.span.outer_str[i]);
        v.push_back(p.span.outer_pk[i]);
    }
    v.push_back((int64_t)p.span_chunks.size());
    for (const auto& c : p.span_chunks) {
        v.insert(v.end(), {c.src, c.pk, c.span, c.plen, c.n, c.body, c.stride, c.perm[0], c.perm[1]});
    }
    v.push_back((int64_t)p.perm_specs.size());
    for (const auto& sp : p.perm_specs) {
        v.insert(v.end(), {sp.W, sp.Dw, sp.ns, sp.pad, (int64_t) reinterpret_cast<uintptr_t>(sp.tab)});
        for (int i = 0; i < 16; ++i) v.push_back(sp.wc[i]);
    }
    v.push_back((int64_t)p.perm_tab.size());
    for (const auto& e : p.perm_tab) v.insert(v.end(), {e.wo4, (int64_t)e.lo, (int64_t)e.hi, (int64_t)e.mix});
    *n = (int64_t)v.size();
    if ((int64_t)v.size() > cap) return fail(MPX_ERR_ARG, "plan dump needs %lld words", (long long)v.size());
    std::copy(v.begin(), v.end(), out);
    return MPX_SUCCESS;
}

int mpx_layout_query(mpx_datatype h, int64_t count, int64_t out[8]) {
    Datatype* d = lookup(h);
    int rc = check_count(count, "count");
    if (rc || (rc = check_usable(d, "query"))) return rc;
    {   // the lowering is host work proportional to the layout: once per count
        std::lock_guard<std::mutex> g(d->mu);
        auto it = d->queries.find(count);
        if (it != d->queries.end()) {
            std::copy(it->second.begin(), it->second.end(), out);
            return MPX_SUCCESS;
        }
    }
    NodeP lay = d->layout_for(count);
    Plan p;
    analyze(lay.get(), &p);
    std::array<int64_t, 8> q = {p.runs, p.nbytes, p.min_off, p.max_end, p.node_count, p.kind, p.overlap,
                                p.kind == PLAN_SPAN ? (int64_t)p.perm_specs.size() : p.chain_align};
    std::copy(q.begin(), q.end(), out);
    std::lock_guard<std::mutex> g(d->mu);
    d->queries.emplace(count, q);
    return MPX_SUCCESS;
}

int mpx_type_iov(mpx_datatype h, int64_t count, int64_t iov_offset, int64_t max_iov_len, int64_t* dev_pairs,
                 int64_t cap_pairs, int64_t* n_out, void* stream) {
    Datatype* d = lookup(h);
    int rc = check_count(count, "count");
    if (rc || (rc = check_usable(d, "query"))) return rc;
    NodeP lay = d->layout_for(count);
    const int64_t total = lay->runs;
    if (iov_offset < 0 || iov_offset > total)  // datatype.py:639-640
        return fail(MPX_ERR_ARG, "iov_offset out of range [0, %lld]", (long long)total);
    if (max_iov_len < -1) return fail(MPX_ERR_ARG, "max_iov_len must be an integer >= -1");
    int64_t n = total - iov_offset;
    if (max_iov_len != -1) n = std::min(n, max_iov_len);
    if (n <= 0) {
        *n_out = 0;
        return MPX_SUCCESS;
    }
    if (n > cap_pairs) return fail(MPX_ERR_ARG, "iov output holds %lld pairs, need %lld",
                                   (long long)cap_pairs, (long long)n);
    int dev = 0;
    if ((rc = device_of(dev_pairs, &dev)) || (rc = ensure_device(dev))) return rc;
    std::string err;
    auto plan = get_plan(d, count, dev, (cudaStream_t)stream, &err);
    if (!plan) return fail(MPX_ERR_OTHER, "%s", err.c_str());
    cudaError_t e = plan_wait(*plan, (cudaStream_t)stream);
    if (e == cudaSuccess) e = launch_iov(*plan, iov_offset, n, dev_pairs, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "iov launch");
    *n_out = n;
    return MPX_SUCCESS;
}

}  // extern "C"

namespace mpx {

// Launch one pack (layout src -> packed dst) or unpack (packed src -> layout
// dst) of limit packed bytes on `stream` of device `dev`.  Either pointer may
// be a peer-device or pinned-host address (the caller enabled access).
int launch_move(int dev, Datatype* d, int64_t count, bool pack, const void* src, void* dst, int64_t limit,
                cudaStream_t stream) {
    if (limit <= 0) return MPX_SUCCESS;
    int rc = ensure_device(dev);
    if (rc) return rc;
    std::string err;
    auto plan = get_plan(d, count, dev, stream, &err);
    if (!plan) return fail(MPX_ERR_OTHER, "%s", err.c_str());
    if (plan->kind == PLAN_EMPTY) return MPX_SUCCESS;
    cudaError_t e = plan_wait(*plan, stream);
    if (e != cudaSuccess) return cuda_fail(e, "descriptor wait");
    if (plan->kind == PLAN_CHAIN && !(!pack && plan->overlap)) {
        ChainBatch b;
        b.njobs = 1;
        ChainJob& j = b.job[0];
        j.c = plan->chain;
        j.src = static_cast<const uint8_t*>(src);
        j.dst = static_cast<uint8_t*>(dst);
        j.limit = limit;
        chain_setup(*plan, pack, &j);
        e = launch_chain_batch(b, pack, dev, stream);
    } else if (plan->kind == PLAN_SPAN && !(!pack && plan->overlap)) {
        e = launch_span(*plan, pack, static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), limit, stream);
    } else if (plan->kind == PLAN_RUNS && !(!pack && plan->overlap)) {
        e = launch_runs(*plan, pack, static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), limit, stream);
    } else {
        e = launch_generic(*plan, pack, static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), limit,
                           stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "pack/unpack launch");
    return MPX_SUCCESS;
}

int launch_zip_move(int dev, Datatype* sd, int64_t scount, const void* src, Datatype* rd, int64_t rcount, void* dst,
                    int64_t bytes, cudaStream_t stream) {
    if (bytes <= 0) return MPX_SUCCESS;
    int rc = ensure_device(dev);
    if (rc) return rc;
    std::string err;
    auto ps = get_plan(sd, scount, dev, stream, &err);
    if (!ps) return fail(MPX_ERR_OTHER, "%s", err.c_str());
    auto pd = get_plan(rd, rcount, dev, stream, &err);
    if (!pd) return fail(MPX_ERR_OTHER, "%s", err.c_str());
    if (ps->kind != PLAN_CHAIN || pd->kind != PLAN_CHAIN || pd->overlap) return MPX_ERR_PENDING;
    cudaError_t e = plan_wait(*ps, stream);
    if (e == cudaSuccess) e = plan_wait(*pd, stream);
    if (e != cudaSuccess) return cuda_fail(e, "descriptor wait");
    e = launch_zip(*ps, *pd, static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), bytes, stream);
    if (e != cudaSuccess) return cuda_fail(e, "zipper launch");
    return MPX_SUCCESS;
}

// contiguous layout_for(count)?  -> offset of its single run
bool contiguous_run(Datatype* d, int64_t count, int64_t* off) {
    NodeP lay = d->layout_for(count);
    if (lay->kind == Kind::Run) {
        *off = lay->off;
        return true;
    }
    return false;
}

int check_layout_region(Datatype* d, int64_t count, int64_t bytes) {
    int rc = check_count(count, "count");
    if (rc || (rc = check_usable(d, "pack/unpack"))) return rc;
    NodeP lay = d->layout_for(count);
    if (lay->runs) {
        if (lay->min_off < 0) return fail(MPX_ERR_ARG, "layout reaches before the start of the buffer");
        if (lay->max_end > bytes)
            return fail(MPX_ERR_ARG, "buffer too small: layout spans %lld bytes, buffer has %lld",
                        (long long)lay->max_end, (long long)bytes);
    }
    return MPX_SUCCESS;
}

int set_device(int dev) { return ensure_device(dev); }

// one pack or unpack, possibly fused with others of the same direction
int movement(int n, const mpx_datatype* dts, const int64_t* counts, const void* const* srcs,
             const int64_t* src_bytes, void* const* dsts, const int64_t* dst_bytes, bool pack,
             cudaStream_t stream, int64_t* written_out) {
    ChainBatch batch;
    batch.njobs = 0;
    int batch_dev = -1;
    bool truncated = false;
    for (int i = 0; i < n; ++i) {
        Datatype* d = lookup(dts[i]);
        std::shared_ptr<Plan> plan;
        int dev = 0;
        const void* layout_buf = pack ? srcs[i] : dsts[i];
        const void* packed_buf = pack ? dsts[i] : srcs[i];
        const int64_t layout_bytes = pack ? src_bytes[i] : dst_bytes[i];
        int rc = prepare(d, counts[i], layout_buf, layout_bytes, packed_buf, stream, &plan, &dev);
        if (rc) return rc;
        const int64_t nbytes = d->size * counts[i];
        int64_t limit = nbytes;
        if (pack) {
            if (dst_bytes[i] < nbytes)
                return fail(MPX_ERR_ARG, "pack output holds %lld bytes, need %lld", (long long)dst_bytes[i],
                            (long long)nbytes);
        } else {
            limit = std::min(src_bytes[i], nbytes);
            if (src_bytes[i] > nbytes) truncated = true;
        }
        if (written_out) written_out[i] = limit;
        if (!plan || limit == 0) continue;
        {
            cudaError_t we = plan_wait(*plan, stream);
            if (we != cudaSuccess) return cuda_fail(we, "descriptor wait");
        }
        const uint8_t* s = static_cast<const uint8_t*>(srcs[i]);
        uint8_t* t = static_cast<uint8_t*>(dsts[i]);
        if (plan->kind == PLAN_CHAIN && !(!pack && plan->overlap)) {
            if (batch.njobs == kMaxJobs || (batch_dev >= 0 && batch_dev != dev)) {
                cudaError_t e = launch_chain_batch(batch, pack, batch_dev, stream);
                if (e != cudaSuccess) return cuda_fail(e, "chain launch");
                batch.njobs = 0;
            }
            ChainJob& j = batch.job[batch.njobs++];
            j.c = plan->chain;
            j.src = s;
            j.dst = t;
            j.limit = limit;
            chain_setup(*plan, pack, &j);
            batch_dev = dev;
        } else if (plan->kind == PLAN_SPAN && !(!pack && plan->overlap)) {
            cudaError_t e = launch_span(*plan, pack, s, t, limit, stream);
            if (e != cudaSuccess) return cuda_fail(e, "span launch");
        } else if (plan->kind == PLAN_RUNS && !(!pack && plan->overlap)) {
            cudaError_t e = launch_runs(*plan, pack, s, t, limit, stream);
            if (e != cudaSuccess) return cuda_fail(e, "run-table launch");
        } else {
            cudaError_t e = launch_generic(*plan, pack, s, t, limit, stream);
            if (e != cudaSuccess) return cuda_fail(e, "generic launch");
        }
    }
    if (batch.njobs) {
        cudaError_t e = launch_chain_batch(batch, pack, batch_dev, stream);
        if (e != cudaSuccess) return cuda_fail(e, "chain launch");
    }
    if (truncated) return fail(MPX_ERR_TRUNCATE, "incoming data larger than the layout");
    return MPX_SUCCESS;
}

}  // namespace mpx

extern "C" {

int mpx_pack(mpx_datatype dt, int64_t count, const void* src, int64_t src_bytes, void* dst, int64_t dst_bytes,
             void* stream) {
    return movement(1, &dt, &count, &src, &src_bytes, &dst, &dst_bytes, true, (cudaStream_t)stream, nullptr);
}

int mpx_unpack(mpx_datatype dt, int64_t count, const void* src, int64_t src_bytes, void* dst, int64_t dst_bytes,
               int64_t* written, void* stream) {
    int64_t w = 0;
    int rc = movement(1, &dt, &count, &src, &src_bytes, &dst, &dst_bytes, false, (cudaStream_t)stream, &w);
    if (written) *written = w;
    return rc;
}

int mpx_pack_multi(int n, const mpx_datatype* dts, const int64_t* counts, const void* const* srcs,
                   const int64_t* src_bytes, void* const* dsts, const int64_t* dst_bytes, void* stream) {
    if (n < 0) return fail(MPX_ERR_ARG, "n must be >= 0");
    return movement(n, dts, counts, srcs, src_bytes, dsts, dst_bytes, true, (cudaStream_t)stream, nullptr);
}

int mpx_unpack_multi(int n, const mpx_datatype* dts, const int64_t* counts, const void* const* srcs,
                     const int64_t* src_bytes, void* const* dsts, const int64_t* dst_bytes, void* stream) {
    if (n < 0) return fail(MPX_ERR_ARG, "n must be >= 0");
    return movement(n, dts, counts, srcs, src_bytes, dsts, dst_bytes, false, (cudaStream_t)stream, nullptr);
}

}  // extern "C"
