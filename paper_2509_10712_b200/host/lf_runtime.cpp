// lf_runtime.cpp -- the two Runtime implementations behind include/loadflow/api.hpp.
//
//  * SimRuntime: deterministic discrete-event engine (reference semantics of
//    proj/src/runtime_virtual.cpp: one actor runs at a time, wake order is
//    (time, schedule sequence), cond waiters wake FIFO, a run with blocked
//    actors and nothing runnable is a deadlock naming the actors, the first
//    actor exception is rethrown from run()).  Implemented as a baton passed
//    between actor threads and the driver under a single engine lock.
//  * WallRuntime: one OS thread per actor on steady_clock with a configurable
//    tick (1 ms = reference realtime runtime, proj/src/runtime_realtime.cpp;
//    1 us = the GPU balancer's clock).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <queue>
#include <sstream>
#include <thread>

#include "loadflow/api.hpp"

namespace loadflow {

namespace {

// ============================================================ simulated time
struct Cancelled {};

class SimRuntime;

struct Actor {
    std::string name;
    std::thread thread;
    std::condition_variable turn;
    bool has_turn = false;
    bool finished = false;
};

struct WakeUp {
    TimeMs at;
    std::uint64_t seq;
    Actor* who;
    bool operator>(const WakeUp& o) const { return at != o.at ? at > o.at : seq > o.seq; }
};

thread_local Actor* t_self = nullptr;

class SimMutex final : public Mutex {
public:
    void lock() override {}    // exclusion is structural: one actor at a time
    void unlock() override {}
};

class SimRuntime final : public Runtime {
public:
    ~SimRuntime() override { shutdown(); }

    TimeMs now() override {
        std::lock_guard<std::mutex> g(m_);
        return clock_;
    }

    void sleep(DurationMs d) override {
        Actor* me = t_self;
        if (me == nullptr) throw std::logic_error("virtual sleep outside actor");
        std::unique_lock<std::mutex> lk(m_);
        enqueue(me, clock_ + std::max<DurationMs>(d, 0));
        park(me, lk);
    }

    void spawn(std::string name, std::function<void()> body) override {
        std::lock_guard<std::mutex> g(m_);
        actors_.push_back(std::make_unique<Actor>());
        Actor* a = actors_.back().get();
        a->name = std::move(name);
        ++alive_;
        enqueue(a, clock_);
        a->thread = std::thread([this, a, body = std::move(body)] {
            t_self = a;
            bool go;
            {
                std::unique_lock<std::mutex> lk(m_);
                go = wait_turn(a, lk);
            }
            if (go) {
                try {
                    body();
                } catch (const Cancelled&) {
                } catch (const std::exception& e) {
                    note_error(a, e.what());
                } catch (...) {
                    note_error(a, "unknown exception");
                }
            }
            std::lock_guard<std::mutex> g2(m_);
            a->finished = true;
            --alive_;
            baton_back_ = true;
            driver_.notify_one();
        });
    }

    void run() override {
        std::unique_lock<std::mutex> lk(m_);
        while (!timeline_.empty() || alive_ > 0) {
            if (timeline_.empty()) {
                std::ostringstream msg;
                msg << "virtual deadlock: " << alive_ << " actor(s) blocked:";
                for (auto& a : actors_)
                    if (!a->finished) msg << " " << a->name;
                lk.unlock();
                shutdown();
                throw std::logic_error(msg.str());
            }
            const WakeUp w = timeline_.top();
            timeline_.pop();
            clock_ = std::max(clock_, w.at);
            baton_back_ = false;
            w.who->has_turn = true;
            w.who->turn.notify_one();
            driver_.wait(lk, [&] { return baton_back_; });
        }
        lk.unlock();
        join_all();
        std::lock_guard<std::mutex> g(m_);
        if (!error_.empty()) throw std::runtime_error("actor failed: " + error_);
    }

    std::unique_ptr<Mutex> make_mutex() override { return std::make_unique<SimMutex>(); }
    std::unique_ptr<Cond> make_cond() override;
    bool is_virtual() const override { return true; }

    // engine internals shared with SimCond (callers hold m_)
    std::mutex m_;
    void enqueue(Actor* a, TimeMs at) { timeline_.push(WakeUp{at, seq_++, a}); }
    TimeMs clock_locked() const { return clock_; }

    // Gives the baton back to the driver and blocks until rescheduled.
    void park(Actor* me, std::unique_lock<std::mutex>& lk) {
        baton_back_ = true;
        driver_.notify_one();
        if (!wait_turn(me, lk)) throw Cancelled{};
    }

private:
    bool wait_turn(Actor* a, std::unique_lock<std::mutex>& lk) {
        a->turn.wait(lk, [&] { return a->has_turn; });
        a->has_turn = false;
        return !cancelled_;
    }

    void note_error(Actor* a, const std::string& what) {
        std::lock_guard<std::mutex> g(m_);
        if (error_.empty()) error_ = a->name + ": " + what;
    }

    void shutdown() {
        {
            std::lock_guard<std::mutex> g(m_);
            cancelled_ = true;
            for (auto& a : actors_) {
                if (a->finished) continue;
                a->has_turn = true;
                a->turn.notify_one();
            }
        }
        join_all();
    }

    void join_all() {
        for (auto& a : actors_)
            if (a->thread.joinable()) a->thread.join();
    }

    std::condition_variable driver_;
    bool baton_back_ = false;
    bool cancelled_ = false;
    TimeMs clock_ = 0;
    std::uint64_t seq_ = 0;
    std::size_t alive_ = 0;
    std::string error_;
    std::priority_queue<WakeUp, std::vector<WakeUp>, std::greater<WakeUp>> timeline_;
    std::vector<std::unique_ptr<Actor>> actors_;
};

class SimCond final : public Cond {
public:
    explicit SimCond(SimRuntime& rt) : rt_(rt) {}

    void wait(Mutex&) override {
        Actor* me = t_self;
        if (me == nullptr) throw std::logic_error("virtual cond wait outside actor");
        std::unique_lock<std::mutex> lk(rt_.m_);
        waiters_.push_back(me);
        rt_.park(me, lk);
    }
    void notify_one() override {
        std::lock_guard<std::mutex> g(rt_.m_);
        if (waiters_.empty()) return;
        rt_.enqueue(waiters_.front(), rt_.clock_locked());
        waiters_.pop_front();
    }
    void notify_all() override {
        std::lock_guard<std::mutex> g(rt_.m_);
        for (Actor* a : waiters_) rt_.enqueue(a, rt_.clock_locked());
        waiters_.clear();
    }

private:
    SimRuntime& rt_;
    std::deque<Actor*> waiters_;   // FIFO: deterministic wake order
};

std::unique_ptr<Cond> SimRuntime::make_cond() { return std::make_unique<SimCond>(*this); }

// ============================================================ wall-clock time
class WallMutex final : public Mutex {
public:
    void lock() override { m_.lock(); }
    void unlock() override { m_.unlock(); }

private:
    std::mutex m_;
};

class WallCond final : public Cond {
public:
    // Mutex is BasicLockable, so condition_variable_any waits on it directly.
    void wait(Mutex& m) override { cv_.wait(m); }
    void notify_one() override { cv_.notify_one(); }
    void notify_all() override { cv_.notify_all(); }

private:
    std::condition_variable_any cv_;
};

class WallRuntime final : public Runtime {
public:
    explicit WallRuntime(std::int64_t tick_ns)
        : tick_(std::chrono::nanoseconds(tick_ns)), t0_(std::chrono::steady_clock::now()) {}

    ~WallRuntime() override {
        for (auto& t : threads_)
            if (t.joinable()) t.join();
    }

    TimeMs now() override { return (std::chrono::steady_clock::now() - t0_) / tick_; }

    void sleep(DurationMs d) override {
        if (d > 0) std::this_thread::sleep_for(d * tick_);
    }

    void spawn(std::string, std::function<void()> body) override {
        std::lock_guard<std::mutex> g(m_);
        ++alive_;
        threads_.emplace_back([this, body = std::move(body)] {
            std::string err;
            try {
                body();
            } catch (const std::exception& e) {
                err = e.what();
            } catch (...) {
                err = "unknown exception";
            }
            std::lock_guard<std::mutex> g2(m_);
            if (!err.empty() && error_.empty()) error_ = err;
            --alive_;
            done_.notify_all();
        });
    }

    void run() override {
        std::vector<std::thread> mine;
        {
            std::unique_lock<std::mutex> lk(m_);
            done_.wait(lk, [&] { return alive_ == 0; });
            mine.swap(threads_);
        }
        for (auto& t : mine)
            if (t.joinable()) t.join();
        std::lock_guard<std::mutex> g(m_);
        if (!error_.empty()) {
            std::string e;
            e.swap(error_);
            throw std::runtime_error("actor failed: " + e);
        }
    }

    std::unique_ptr<Mutex> make_mutex() override { return std::make_unique<WallMutex>(); }
    std::unique_ptr<Cond> make_cond() override { return std::make_unique<WallCond>(); }
    bool is_virtual() const override { return false; }
    std::int64_t tick_ns() const override { return tick_.count(); }

private:
    std::chrono::nanoseconds tick_;
    std::chrono::steady_clock::time_point t0_;
    std::mutex m_;
    std::condition_variable done_;
    std::vector<std::thread> threads_;
    std::size_t alive_ = 0;
    std::string error_;
};

}  // namespace

std::unique_ptr<Runtime> make_virtual_runtime() { return std::make_unique<SimRuntime>(); }
std::unique_ptr<Runtime> make_realtime_runtime() { return std::make_unique<WallRuntime>(1'000'000); }
std::unique_ptr<Runtime> make_realtime_runtime_ticks(std::int64_t tick_ns) {
    if (tick_ns < 1) throw std::invalid_argument("tick must be >= 1 ns");
    return std::make_unique<WallRuntime>(tick_ns);
}

}  // namespace loadflow
