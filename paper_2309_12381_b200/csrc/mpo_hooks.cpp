// mpo_hooks.cpp -- native post-accumulate-grad hooks of the fused backward ("operate the
// optimization step as soon as the gradient is computed ... the gradient is then not needed
// anymore").  The paper's per-parameter step costs one Python call per parameter when the hook is
// a Python function; at short backwards (GPT-2, B=1, T=128) that host time is most of the
// overhead.  Here the hook is a C++ torch::autograd::PostAccumulateGradHook installed in each
// parameter's autograd slot: it builds the parameter's hyper-parameter struct, calls the C ABI
// (mpo_fused_backward_hook_step, or one mpo_adam_step / mpo_sgd_step over the batched small
// parameters at the end of backward) on the current CUDA stream and frees the gradient.
//
// Plumbing only: every number is computed by libmpo's kernels (include/mpo.h), whose entry points
// arrive as function pointers of the library the Python side loaded (exact or FMA build).  The
// optimizer's Python object keeps the residual / m / v tensors alive and disarms this state when
// it is collected (the hooks then do nothing).
#include <torch/extension.h>
#include <torch/csrc/autograd/engine.h>
#include <torch/csrc/autograd/function_hook.h>
#include <torch/csrc/autograd/variable.h>
#include <c10/cuda/CUDAStream.h>
#include <cuda_runtime_api.h>

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mpo.h"

namespace {

using HookFn = mpo_status (*)(mpo_optim, mpo_dtype, mpo_dtype, const mpo_tensor*, const void*, double*, mpo_stream);
using AdamFn = mpo_status (*)(mpo_dtype, mpo_dtype, const mpo_tensor*, int32_t, const mpo_adam_hp*, int32_t, double*,
                              mpo_stream);
using SgdFn = mpo_status (*)(mpo_dtype, mpo_dtype, const mpo_tensor*, int32_t, const mpo_sgd_hp*, int32_t, double*,
                             mpo_stream);
using ErrFn = const char* (*)();

// the per-step key of the stochastic-rounding draws (same mixing as api.step_seed)
inline uint64_t step_seed(uint64_t seed, int64_t step) { return seed * 0x9E3779B97F4A7C15ull + uint64_t(step); }

int grad_code(at::ScalarType t) {
    switch (t) {
        case at::kHalf: return MPO_FP16;
        case at::kBFloat16: return MPO_BF16;
        case at::kFloat: return MPO_FP32;
        default: throw std::runtime_error("mpo hook: unsupported gradient dtype (fp16, bf16 or fp32)");
    }
}

struct Param {
    mpo_tensor row;   // value / resid / m / v / n / sr_stream; grad filled per call
    int group = 0;
    int vdt = 0;      // storage format code of the value
    int64_t* step = nullptr;   // this parameter's count in the optimizer's shared int64 buffer
};

class HookState : public std::enable_shared_from_this<HookState> {
   public:
    HookState(int kind, uint64_t seed, int64_t batch_below, int64_t flush_elems, int64_t steps, int64_t hook_fn,
              int64_t adam_fn, int64_t sgd_fn, int64_t err_fn, int64_t norm_ws, int64_t hook_S, int64_t host_S)
        : kind_(kind), seed_(seed), batch_below_(batch_below), flush_elems_(flush_elems),
          steps_(reinterpret_cast<int64_t*>(steps)),
          hook_fn_(reinterpret_cast<HookFn>(hook_fn)), adam_fn_(reinterpret_cast<AdamFn>(adam_fn)),
          sgd_fn_(reinterpret_cast<SgdFn>(sgd_fn)), err_fn_(reinterpret_cast<ErrFn>(err_fn)),
          norm_ws_(reinterpret_cast<double*>(norm_ws)), hook_S_(reinterpret_cast<double*>(hook_S)),
          host_S_(reinterpret_cast<double*>(host_S)) {
        if (hook_S_ && cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming) != cudaSuccess)
            throw std::runtime_error("mpo hook: cudaEventCreate failed");
    }
    ~HookState() {
        if (ev_) cudaEventDestroy(ev_);
    }

    // sr_stream = the parameter's index: its slot in the step-count buffer and in hook_S
    int add_param(int64_t value, int64_t resid, int64_t m, int64_t v, int64_t n, int32_t sr_stream, int group,
                  int vdt) {
        Param p;
        std::memset(&p.row, 0, sizeof(p.row));
        p.row.value = reinterpret_cast<void*>(value);
        p.row.resid = reinterpret_cast<void*>(resid);
        p.row.m = reinterpret_cast<float*>(m);
        p.row.v = reinterpret_cast<float*>(v);
        p.row.n = n;
        p.row.sr_stream = sr_stream;
        p.group = group;
        p.vdt = vdt;
        p.step = steps_ + sr_stream;
        params_.push_back(p);
        return int(params_.size()) - 1;
    }

    // the hyper-parameters of a param group as the raw bytes of an mpo_adam_hp / mpo_sgd_hp
    void set_group(int gi, const std::string& bytes) {
        const size_t want = kind_ == MPO_ADAM ? sizeof(mpo_adam_hp) : sizeof(mpo_sgd_hp);
        if (bytes.size() != want) throw std::runtime_error("mpo hook: hyper-parameter struct size mismatch");
        if (gi < 0) throw std::runtime_error("mpo hook: negative group");
        if (size_t(gi) >= groups_.size()) groups_.resize(size_t(gi) + 1);
        groups_[size_t(gi)] = bytes;
    }

    void disarm() { alive_ = false; }
    int64_t calls() const { return calls_; }

    // skip_nonfinite: roll back the step counts of the parameters whose update the last backward
    // skipped (their S reached the host through the copy queued at its end)
    void resolve() {
        std::lock_guard<std::recursive_mutex> lk(mu_);
        if (!check_pending_) return;
        check_pending_ = false;
        if (cudaEventSynchronize(ev_) != cudaSuccess) throw std::runtime_error("mpo hook: cudaEventSynchronize failed");
        for (size_t i = 0; i < params_.size(); ++i)
            if (!std::isfinite(host_S_[i])) *params_[i].step -= 1;
    }

    void on_grad(int idx, const at::Tensor& t) {
        // parameters on several devices: the engine may run their hooks from several device threads
        std::lock_guard<std::recursive_mutex> lk(mu_);
        if (!alive_) return;
        at::Tensor& g = t.mutable_grad();
        if (!g.defined()) return;
        if (check_pending_) resolve();
        Param& p = params_[size_t(idx)];
        *p.step += 1;
        if (!g.is_cuda() || !g.is_contiguous()) throw std::runtime_error("mpo hook: gradient must be a contiguous CUDA tensor");
        if (p.row.n < batch_below_) {
            // small parameters (biases, norms): held until one multi-tensor launch at the end of
            // backward or once flush_elems are pending
            pending_.emplace_back(idx, g);
            pending_elems_ += p.row.n;
            g = at::Tensor();
            queue_flush();
            if (pending_elems_ >= flush_elems_) flush(false);
            return;
        }
        const int gdt = grad_code(g.scalar_type());
        mpo_tensor row = p.row;
        row.grad = g.data_ptr();
        row.hp = 0;
        cudaStream_t s = c10::cuda::getCurrentCUDAStream(g.device().index()).stream();
        mpo_status st;
        if (kind_ == MPO_ADAM) {
            mpo_adam_hp hp = adam_hp(p);
            st = hook_fn_(MPO_ADAM, mpo_dtype(p.vdt), mpo_dtype(gdt), &row, &hp, norm_ws_, s);
        } else {
            mpo_sgd_hp hp = sgd_hp(p);
            st = hook_fn_(MPO_SGD, mpo_dtype(p.vdt), mpo_dtype(gdt), &row, &hp, norm_ws_, s);
        }
        if (st != MPO_OK) throw std::runtime_error(std::string("mpo_fused_backward_hook_step: ") + err_fn_());
        ++calls_;
        if (hook_S_) {
            // this parameter's S (norm_ws[0] of its call) for the step-count rollback of a skip
            if (cudaMemcpyAsync(hook_S_ + row.sr_stream, norm_ws_, sizeof(double), cudaMemcpyDeviceToDevice, s) !=
                cudaSuccess)
                throw std::runtime_error("mpo hook: cudaMemcpyAsync failed");
            queue_flush();
        }
        g = at::Tensor();   // freed now; stream order makes the block's reuse safe
    }

    void flush(bool final) {
        std::lock_guard<std::recursive_mutex> lk(mu_);
        if (final) flush_queued_ = false;
        if (!pending_.empty()) launch_pending();
        if (final && hook_S_ && alive_) {
            cudaStream_t s = c10::cuda::getCurrentCUDAStream().stream();
            const size_t bytes = params_.size() * sizeof(double);
            if (cudaMemcpyAsync(host_S_, hook_S_, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaMemsetAsync(hook_S_, 0, bytes, s) != cudaSuccess || cudaEventRecord(ev_, s) != cudaSuccess)
                throw std::runtime_error("mpo hook: end-of-backward found-inf copy failed");
            check_pending_ = true;
        }
    }

   private:
    mpo_adam_hp adam_hp(const Param& p) const {
        mpo_adam_hp hp;
        std::memcpy(&hp, groups_.at(size_t(p.group)).data(), sizeof(hp));
        hp.step = *p.step;
        hp.seed = step_seed(seed_, *p.step);
        return hp;
    }
    mpo_sgd_hp sgd_hp(const Param& p) const {
        mpo_sgd_hp hp;
        std::memcpy(&hp, groups_.at(size_t(p.group)).data(), sizeof(hp));
        hp.first_step = *p.step == 1;
        hp.seed = step_seed(seed_, *p.step);
        return hp;
    }

    void queue_flush() {
        if (flush_queued_) return;
        flush_queued_ = true;
        std::weak_ptr<HookState> w = shared_from_this();
        torch::autograd::Engine::get_default_engine().queue_callback([w] {
            if (auto s = w.lock()) s->flush(true);
        });
    }

    void launch_pending() {
        std::vector<std::pair<int, at::Tensor>> pending;
        pending.swap(pending_);
        pending_elems_ = 0;
        // one launch per (value format, gradient dtype); hyper-parameter groups per (group, step)
        std::map<std::pair<int, int>, std::vector<size_t>> by_dtype;
        for (size_t k = 0; k < pending.size(); ++k)
            by_dtype[{params_[size_t(pending[k].first)].vdt, grad_code(pending[k].second.scalar_type())}].push_back(k);
        cudaStream_t s = c10::cuda::getCurrentCUDAStream(pending[0].second.device().index()).stream();
        for (auto& kv : by_dtype) {
            std::vector<mpo_tensor> rows;
            std::map<std::pair<int, int64_t>, int> keys;
            std::vector<mpo_adam_hp> ahp;
            std::vector<mpo_sgd_hp> shp;
            for (size_t k : kv.second) {
                const Param& p = params_[size_t(pending[k].first)];
                auto key = std::make_pair(p.group, *p.step);
                auto it = keys.find(key);
                int h;
                if (it == keys.end()) {
                    h = int(keys.size());
                    keys[key] = h;
                    if (kind_ == MPO_ADAM) ahp.push_back(adam_hp(p));
                    else shp.push_back(sgd_hp(p));
                } else {
                    h = it->second;
                }
                mpo_tensor row = p.row;
                row.grad = pending[k].second.data_ptr();
                row.hp = h;
                rows.push_back(row);
            }
            // one launch per MPO_MAX_HP_GROUPS (group, step) pairs (a launch's hyper-parameter bank)
            const int nk = int(keys.size());
            for (int c = 0; c < nk; c += MPO_MAX_HP_GROUPS) {
                const int ce = c + MPO_MAX_HP_GROUPS < nk ? c + MPO_MAX_HP_GROUPS : nk;
                std::vector<mpo_tensor> sub;
                for (const mpo_tensor& r : rows)
                    if (r.hp >= c && r.hp < ce) {
                        sub.push_back(r);
                        sub.back().hp = r.hp - c;
                    }
                mpo_status st = kind_ == MPO_ADAM
                                    ? adam_fn_(mpo_dtype(kv.first.first), mpo_dtype(kv.first.second), sub.data(),
                                               int32_t(sub.size()), ahp.data() + c, int32_t(ce - c), nullptr, s)
                                    : sgd_fn_(mpo_dtype(kv.first.first), mpo_dtype(kv.first.second), sub.data(),
                                              int32_t(sub.size()), shp.data() + c, int32_t(ce - c), nullptr, s);
                if (st != MPO_OK) throw std::runtime_error(std::string("mpo step (batched hook flush): ") + err_fn_());
                ++calls_;
            }
        }
        // the gradients are released here (stream order keeps their reuse safe)
    }

    std::recursive_mutex mu_;   // on_grad -> flush / resolve re-enter it on the same thread
    int kind_;
    uint64_t seed_;
    int64_t batch_below_, flush_elems_;
    int64_t* steps_;
    HookFn hook_fn_;
    AdamFn adam_fn_;
    SgdFn sgd_fn_;
    ErrFn err_fn_;
    double* norm_ws_;
    double* hook_S_;
    double* host_S_;
    cudaEvent_t ev_ = nullptr;
    bool check_pending_ = false;
    bool alive_ = true;
    bool flush_queued_ = false;
    int64_t calls_ = 0;
    std::vector<Param> params_;
    std::vector<std::string> groups_;
    std::vector<std::pair<int, at::Tensor>> pending_;
    int64_t pending_elems_ = 0;
};

struct MpoHook : torch::autograd::PostAccumulateGradHook {
    MpoHook(std::shared_ptr<HookState> st, int idx) : st_(std::move(st)), idx_(idx) {}
    void operator()(const torch::autograd::Variable& tensor) override { st_->on_grad(idx_, tensor); }
    std::shared_ptr<HookState> st_;
    int idx_;
};

void install(const std::shared_ptr<HookState>& st, const at::Tensor& param, int idx) {
    if (!param.requires_grad() || !param.is_leaf()) throw std::runtime_error("mpo hook: parameter must be a leaf that requires grad");
    if (torch::autograd::impl::post_acc_grad_hooks(param))
        throw std::runtime_error("mpo hook: the parameter already has post-accumulate-grad hooks");
    torch::autograd::impl::set_post_acc_grad_hooks(param, std::make_unique<MpoHook>(st, idx));
}

void uninstall(const at::Tensor& param) { torch::autograd::impl::set_post_acc_grad_hooks(param, nullptr); }

}  // namespace

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
    m.doc() = "native post-accumulate-grad hooks of the fused backward step (calls the libmpo C ABI)";
    py::class_<HookState, std::shared_ptr<HookState>>(m, "HookState")
        .def(py::init<int, uint64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                      int64_t, int64_t>())
        .def("add_param", &HookState::add_param)
        .def("set_group", [](HookState& s, int gi, py::bytes b) { s.set_group(gi, std::string(b)); })
        .def("resolve", &HookState::resolve)
        .def("disarm", &HookState::disarm)
        .def("calls", &HookState::calls);
    m.def("install", &install);
    m.def("uninstall", &uninstall);
}
